// htrise-b200 device kernels: declarations shared by the launch sites.
//
// All kernels are f64 and deterministic (fixed reduction trees, no FP64
// atomics): every rank of a sharded run computes bit-identical results from
// bit-identical inputs, which keeps the redundant per-rank eigen-truncations
// in lock-step.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <mutex>
#include <map>
#include <utility>

namespace htr {

constexpr int kNumSMs = 148;  // B200; the launchers query the device anyway

/// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
/// current device. The attribute is per (function, device); the largest
/// value applied so far is remembered per pair under a lock and the limit
/// only ever grows (it is never rewritten while launches of the kernel may
/// be in flight), so contexts on several devices and concurrent callers each
/// configure what they launch.
inline cudaError_t ensure_smem_limit(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> applied;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = applied[std::make_pair(fn, dev)];
    if (bytes <= cur) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e == cudaSuccess) cur = bytes;
    return e;
}

// ---------------------------------------------------------------------------
// Generic strided contraction ("mode product engine").
//   C(m, n1, n2) = alpha * sum_{k1<K1, k2<K2} A(m, k1, k2) * B(k1, k2, n1, n2)
//                  + beta * C(m, n1, n2)
// Offsets: A = m*sam + k1*sak1 + k2*sak2, B = k1*sbk1 + k2*sbk2 + n1*sbn1 +
// n2*sbn2, C = m*scm + n1*scn1 + n2*scn2 (+ batch * sab/sbb/scb); N and K
// must stay below 2^31. Covers every mode product (leaf
// projection U^T, reconstruction U, transfer split) and every mode-k Gram
// Y_(k) Y_(k)^T of a canonical tensor without materialising an unfolding.
// ---------------------------------------------------------------------------
struct GemmDesc {
    int64_t M = 1, N1 = 1, N2 = 1, K1 = 1, K2 = 1;
    int64_t batch = 1;                   // independent problems, pointer strides below
    int64_t sab = 0, sbb = 0, scb = 0;
    const double* A = nullptr;
    int64_t sam = 0, sak1 = 0, sak2 = 0;
    const double* B = nullptr;
    int64_t sbk1 = 0, sbk2 = 0, sbn1 = 0, sbn2 = 0;
    double* C = nullptr;
    int64_t scm = 0, scn1 = 0, scn2 = 0;
    double alpha = 1.0, beta = 0.0;
    // residual-energy epilogue: instead of storing, accumulate
    // sum (D(m,n) - acc)^2 with D addressed like C; one partial per CTA.
    const double* D = nullptr;
    double* energy_partials = nullptr;  // >= grid size entries
    // C = A A^T-like symmetric result (M == N, C column- or row-major square):
    // on the fast kernel only the tiles touching the lower triangle are
    // computed and the strict upper triangle is mirrored from it afterwards
    // (ignored, i.e. everything computed, on the general kernel)
    bool symmetric = false;
};

// Enqueue; returns the number of CTAs used for the energy epilogue (0 when
// storing). `workspace` must hold gemm_workspace_doubles(desc) doubles.
int64_t gemm_workspace_doubles(const GemmDesc& d, int num_sms);
// Number of per-CTA partials the residual-energy epilogue writes.
int64_t gemm_energy_partials(const GemmDesc& d, int num_sms);
// With sq_partials (plain-store GEMMs on the fast path only) every CTA also
// writes the sum of squares of the outputs it stored; gemm_energy_partials()
// entries. Callers check gemm_is_fast() first.
int launch_gemm(const GemmDesc& d, double* workspace, int num_sms, cudaStream_t s, int64_t* launches,
                double* sq_partials = nullptr);
bool gemm_is_fast(const GemmDesc& d, int num_sms);
// out[i + I (q + Q o)] = sum_j M(q, j) t[i + I (j + J o)], M(q, j) =
// M[q*smq + j*smj]: the r -> n expansions of decode (J <= 32, Q <= 128, I
// even, 16-byte aligned t and out). Persistent DMMA kernel with M resident
// in shared memory. Returns the CTA count, or -1 when not applicable.
int launch_expand(const double* t, int64_t I, int64_t J, int64_t O, const double* M, int64_t Q, int64_t smq,
                  int64_t smj, double* out, int num_sms, cudaStream_t s, int64_t* launches);

// Sum of squares of n doubles -> out[0] (deterministic two-pass). partials
// needs kReduceBlocks doubles. Also writes out[1] = 1.0 if any entry is
// non-finite, else 0.0.
constexpr int kReduceBlocks = 592;
void launch_sumsq(const double* x, int64_t n, double* partials, double* out, cudaStream_t s,
                  int64_t* launches);
// out[0] = sum of n partials in index order (deterministic).
void launch_sum_partials(const double* partials, int64_t n, double* out, cudaStream_t s, int64_t* launches);

constexpr int64_t kJacobiMaxN = 2048;  // largest Gram the device eigensolver takes
// Symmetric eigen-decomposition of an n x n column-major matrix G by
// parallel cyclic Jacobi in one CTA. Writes eigenvalues (descending) to
// lambda and the matching eigenvectors as columns of V (n x n, col-major).
// `work` must hold 2*n*n doubles when n exceeds the shared-memory limit.
/// Eigenproblems the batched one-CTA solver takes (n <= 135).
bool jacobi_batchable(int64_t n);
/// Independent symmetric eigenproblems, one CTA each, side by side; each
/// result equals launch_jacobi_eig's bit for bit. Every n must be batchable.
void launch_jacobi_eig_batch(const double* const* G, const int64_t* n, double* const* lambda, double* const* V,
                             int count, cudaStream_t s, int64_t* launches);
void launch_jacobi_eig(const double* G, int64_t n, double* lambda, double* V, double* work, cudaStream_t s,
                       int64_t* launches);

// Tridiagonal route of the symmetric eigen-truncation (k_tridiag.cu), for
// 1 <= n <= 1024: launch_tridiag_eigvals reduces each G_i (n_i x n_i,
// symmetric) to tridiagonal form in workspace W_i
// (tridiag_workspace_doubles(n_i)) and writes all its eigenvalues, descending,
// to lambda_i; launch_tridiag_vectors then writes the r_i leading
// eigenvectors to U_i (n_i x r_i, orthonormal), or identity columns when
// info_i[2] == 0 (the rank rule's zero-input flag). One CTA per problem.
bool tridiag_supported(int64_t n);
constexpr int64_t kTriFullMaxN = 64;  // all n eigenvectors by inverse iteration up to this size
int64_t tridiag_workspace_doubles(int64_t n);
void launch_tridiag_eigvals(const double* const* G, const int64_t* n, double* const* lambda, double* const* W,
                            int count, cudaStream_t s, int64_t* launches);
void launch_tridiag_vectors(const double* const* W, const double* const* info, const int64_t* n, const int64_t* r,
                            double* const* U, int count, cudaStream_t s, int64_t* launches);

// flag[0] = 1 if G - shift I (n x n, symmetric) is positive definite (one-CTA
// Cholesky on `work`, n * n doubles), else 0.
void launch_posdef_test(const double* G, int64_t n, double shift, double* work, double* flag, cudaStream_t s,
                        int64_t* launches);

// Blocked form of the positive-definiteness test: launch_chol_prepare writes
// A = G - shift I (n x n) and flag[0] = 1; launch_chol_panel factors the
// columns [kb, kb + b) (b = 32 except for the last panel) of the current
// trailing matrix, clearing flag[0] on a non-positive pivot; the caller
// applies A[kb+b:, kb+b:] -= P P^T (P = A[kb+b:, kb:kb+b]) between panels.
constexpr int64_t kCholPanel = 32;
void launch_chol_prepare(const double* G, int64_t n, double shift, double* A, double* flag, cudaStream_t s,
                         int64_t* launches);
void launch_chol_panel(double* A, int64_t n, int64_t kb, int64_t b, double* flag, cudaStream_t s, int64_t* launches);

// Rank rule of truncated_svd.hpp:74-99 on k = min(rows, cols) values
// sigma_i^2 = max(lambda_i, 0). info[0] = rank, info[1] = discarded norm,
// info[2] = trace (sum of lambda) used for the zero-input test.
void launch_rank_rule(const double* lambda, int64_t k, int64_t n, double eps_abs, int64_t min_rank,
                      const double* trace_src, double* info, cudaStream_t s, int64_t* launches);

// Copy the first r columns of V (n x n) to U (n x r); when zero_input != 0
// writes identity columns instead (truncated_svd.hpp:66-72).
void launch_take_columns(const double* V, int64_t n, int64_t r, double* U, const double* info,
                         cudaStream_t s, int64_t* launches);

// dst (outer x (a_ext+extra) x inner-block) <- zero-padded copy along one axis:
// src viewed as [inner, ext, outer] -> dst [inner, ext+extra, outer].
void launch_pad_axis(const double* src, int64_t inner, int64_t ext, int64_t outer, int64_t extra, double* dst,
                     cudaStream_t s, int64_t* launches);

// dst (ext x inner*outer, col-major) <- the unfolding of src viewed as
// [inner, ext, outer] along its middle axis.
void launch_unfold(const double* src, int64_t inner, int64_t ext, int64_t outer, double* dst, cudaStream_t s,
                   int64_t* launches);

// Orthogonalise W (alpha x q) against U (alpha x r) twice, then CholeskyQR2,
// in one CTA (ht_rise.hpp:53-79 expand_core with SURVEY §7.3 item 4). Writes
// the orthonormal result back into W and the defect ||U^T W||_F, ||W||_F to
// info[0..1].
void launch_orthonormalize_new(const double* U, int64_t alpha, int64_t r, double* W, int64_t q, double* info,
                               double* work, cudaStream_t s, int64_t* launches);

// Per-field statistics of x (n elements; field of flat index e is
// (e / inner) % F): kind 0 max |v|, 1 sum v^2, 2 sum v, 3 sum (v - mu[f])^2;
// out[f] for every field (deterministic: fixed per-CTA and cross-CTA
// orders). partials: field_stat_blocks(num_sms) * 16 doubles.
int field_stat_blocks(int num_sms);
void launch_field_stat(const double* x, int64_t n, int64_t inner, int F, int kind, const double* mu, double* partials,
                       double* out, int num_sms, cudaStream_t s, int64_t* launches);
// out = (x - mu[f]) / sc[f], or with `inverse` out = x * sc[f] + mu[f]
// (mu may be null: 0).
void launch_field_apply(const double* x, int64_t n, int64_t inner, int F, const double* mu, const double* sc,
                        bool inverse, double* out, int num_sms, cudaStream_t s, int64_t* launches);

// dst = src with its axes permuted: output mode k is input mode perm[k]
// (d <= 16, canonical layouts).
void launch_permute(const double* src, const int64_t* shape, int d, const int64_t* perm, double* dst, cudaStream_t s,
                    int64_t* launches);

// Orthonormality defects of `count` bases U_i (alpha_i x r_i, col-major):
// out[i] = ||U_i^T U_i - I||_F, one CTA per basis (r_i = 0 writes 0).
void launch_basis_defect(const double* const* U, const int64_t* alpha, const int64_t* r, int count, double* out,
                         cudaStream_t s, int64_t* launches);

// out[i, q, o] = sum_j M(q, j) t[i, j, o] with M(q, j) = M[q*smq + j*smj],
// J, Q <= 32 (streaming, one thread per fibre). When energy != nullptr the
// kernel also writes per-CTA partials of sum ||t_fibre - M^T (M t_fibre)||^2,
// and with ysq != nullptr per-CTA partials of ||t||^2 (the input is read once
// for all three). Both partial arrays need 8 * num_sms entries. Returns the
// CTA count, or -1 when the extents are too large.
int launch_mode_small(const double* t, int64_t I, int64_t J, int64_t O, const double* M, int64_t Q, int64_t smq,
                      int64_t smj, double* out, double* energy, double* ysq, int num_sms, cudaStream_t s,
                      int64_t* launches);

// Two adjacent modes at once (t viewed as [I, J0, J1, O] -> out [I, Q0, Q1, O]):
// out = t x_0 U0^T x_1 U1^T with U0 J0 x Q0, U1 J1 x Q1 (column-major bases),
// J <= 8, Q <= 4; per-CTA ||t||^2 partials in ysq (8 * num_sms entries) when
// given. Returns the CTA count, or -1 when the extents are out of range.
int launch_pair_project(const double* t, int64_t I, int64_t J0, int64_t J1, int64_t O, const double* U0, int64_t Q0,
                        const double* U1, int64_t Q1, double* out, double* ysq, int num_sms, cudaStream_t s,
                        int64_t* launches);

// Fill dst[i] = value for n entries.
void launch_fill(double* dst, int64_t n, double value, cudaStream_t s, int64_t* launches);

// Fused all-leaf projection for 3-way batches [N0, N1, n2, S] on the FP64
// tensor cores (DMMA): Z[a0,a1,a2,s] = sum X[i0,i1,i2,s] U0[i0,a0] U1[i1,a1]
// U2[i2,a2] and sum X^2, in one read of X (K1). Enqueues the
// streaming kernel plus the small slab-axis contraction GEMM.
struct Fused3Args {
    const double* Y = nullptr;
    int64_t n2 = 0, S = 0;
    const double* U0 = nullptr;  // N0 x r0
    const double* U1 = nullptr;  // N1 x r1
    const double* U2 = nullptr;  // n2 x r2
    int r0 = 0, r1 = 0, r2 = 0;
    double* Z = nullptr;          // r0*r1*r2 x S
    double* wslab = nullptr;      // workspace: per-slab W (r0 r1 per slab)
    double* ysq_partials = nullptr;  // grid entries
    double* wpart = nullptr;      // split-slab partial W (set by the launcher, after ysq_partials)
    bool slab_gemm = true;        // also enqueue Z = sum_i2 W (x) U2 (else left to tail3)
};
// Whether the fused kernel supports this shape; returns the grid size used.
bool fused3_supported(int64_t n0, int64_t n1, int64_t n2, int r0, int r1, int r2);
int64_t fused3_workspace_doubles(int64_t n0, int64_t n1, int64_t n2, int64_t S, int r0, int r1, int r2,
                                 int num_sms);
int launch_fused3(int64_t n0, int64_t n1, const Fused3Args& a, int num_sms, cudaStream_t s, int64_t* launches);

// Skip-path tail for (1,(2,3)) trees, one CTA per sample: Z_s from the
// per-slab W of fused3 and U2, then latent_s = Z_s B (B: r1 r2 x rt transfer
// basis), latent [r0, rt, S] and ||latent_s||^2 per sample.
struct Tail3Args {
    const double* wslab = nullptr;
    const double* U2 = nullptr;
    const double* B = nullptr;
    int r0 = 0, r1 = 0, r2 = 0, rt = 0;
    int64_t n2 = 0, S = 0;
    double* latent = nullptr;
    double* latsq = nullptr;  // S entries
    // final reductions, done by the last CTA to finish (fixed order):
    // out[0] = sum(ysq_partials[0..n_ysq)), out[2] = sum(latsq[0..S))
    const double* ysq_partials = nullptr;
    int64_t n_ysq = 0;
    double* out = nullptr;
    // optional copy of out[0] / out[2] in mapped pinned host memory (the host
    // reads it after the stream or an event completes: no D2H copy)
    double* host_out = nullptr;
    unsigned int* ticket = nullptr;  // zero on entry, left zero on exit
    int variant = 0;  // 0 auto, 1 one sample per CTA, 2 sample pairs (falls back to 1 when it does not fit)
    int num_sms = kNumSMs;
    int csize = 1;    // CTAs per sample (a thread-block cluster), set by the launcher
    bool identity_transfer = false;  // B == I (rt == r1 r2): latent = Z, no projection
};
bool tail3_supported(int r0, int r1, int r2, int rt, int64_t n2);
/// Entries the tail writes into Tail3Args::latsq (whichever kernel it picks).
int64_t tail3_latsq_entries(int64_t S, int num_sms);

// Skip-path tail for balanced 4-way trees ((1,2),(3,4)), one CTA per sample
// (k_tail4.cu): from fused3's per-slab W = [R01 = r0 r1, n2, n3, S] to the
// latent [r12, r34, S] through B12 (R01 x r12), U2 (n2 x r2), U3 (n3 x r3)
// and B34 (r2 r3 x r34), with ||latent_s||^2 and the final scalar reductions
// as in Tail3Args.
struct Tail4Args {
    const double* W = nullptr;
    const double* B12 = nullptr;
    const double* U2 = nullptr;
    const double* U3 = nullptr;
    const double* B34 = nullptr;
    int R01 = 0, r12 = 0, r2 = 0, r3 = 0, r34 = 0;
    int64_t n2 = 0, n3 = 0, S = 0;
    double* latent = nullptr;
    double* latsq = nullptr;  // S entries
    const double* ysq_partials = nullptr;
    int64_t n_ysq = 0;
    double* out = nullptr;
    double* host_out = nullptr;
    unsigned int* ticket = nullptr;  // zero on entry, left zero on exit
    int csize = 1;  // CTAs per sample (a thread-block cluster over the i3 slices), set by the launcher
};
bool tail4_supported(int R01, int r12, int r34, int r2, int r3, int64_t n2, int64_t n3);
void launch_tail4(const Tail4Args& a, int num_sms, cudaStream_t s, int64_t* launches);
// (identity_transfer is honoured by the per-sample/cluster kernel; the
// sample-pair variant falls back to it)

// Balanced 4-leaf subtree over 4 consecutive modes of extent 8, all ranks 4
// (config 4): every contiguous 8^4 block o of X (O blocks, 16-byte aligned)
// -> the subtree root's 4 outputs out[(o % P) + P (c + 4 (o / P))], through
// the 4 leaf projections and the 3 transfers. The first launch over y writes
// per-CTA ||y||^2 partials; the finishing launch writes per-CTA ||out||^2
// partials and its last CTA sc[0] = ||y||^2, sc[2] = ||out||^2.
struct QuadArgs {
    const double* X = nullptr;
    int64_t O = 0, P = 1;
    const double* U[4] = {nullptr, nullptr, nullptr, nullptr};  // 8 x 4 leaf bases
    const double* T01 = nullptr;  // 16 x 4 basis of the transfer over leaves 0,1
    const double* T23 = nullptr;  // leaves 2,3
    const double* T = nullptr;    // the subtree root (over the two transfers)
    double* out = nullptr;
    double* partials = nullptr;   // >= grid entries
    const double* ysq_partials = nullptr;  // finishing launch: the first launch's partials
    int64_t n_ysq = 0;
    double* sc = nullptr;
    double* host_out = nullptr;
    unsigned int* ticket = nullptr;
};
/// Two adjacent modes projected in one read (k_proj2.cu): Y viewed as
/// [n0, n1, n2, S] -> C[n0, r1, r2, S] = Y x_1 U1^T x_2 U2^T (U1 n1 x r1,
/// U2 n2 x r2, column-major). n0 % 8 == 0, n1 % 4 == 0, n1 <= 256, r <= 24.
struct Proj2Args {
    const double* Y = nullptr;
    int64_t n0 = 0, n1 = 0, n2 = 0, S = 0;
    const double* U1 = nullptr;
    const double* U2 = nullptr;
    int r1 = 0, r2 = 0;
    double* C = nullptr;
};
bool proj2_supported(const Proj2Args& a);
int launch_proj2(const Proj2Args& a, cudaStream_t s, int64_t* launches);
/// Streaming Gram G = Y_(k) Y_(k)^T of Y viewed as [K, M, B] (K contiguous,
/// M <= 128, K even; k_gram.cu). partials: gram_stream_partials doubles.
bool gram_stream_supported(const double* Y, int64_t K, int64_t M, int64_t B);
int64_t gram_stream_partials(int64_t M, int num_sms);
int launch_gram_stream(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                       cudaStream_t s, int64_t* launches);
/// The Gram of mode 0 (X = [M, C], rows contiguous, M even, M <= 128) on
/// DMMA from shared-memory column chunks; partials: gram_stream_partials(M).
bool gram_mode0_supported(const double* X, int64_t M, int64_t C);
int launch_gram_mode0(const double* X, int64_t M, int64_t C, double* partials, double* G, int num_sms, cudaStream_t s,
                      int64_t* launches);
/// The same Gram for 9 <= M <= 32 rows (any K >= 1, incl. mode 0) on DMMA,
/// four columns per k-step. partials: gram_mid_partials doubles.
bool gram_mid_supported(int64_t K, int64_t M, int64_t B);
int64_t gram_mid_partials(int num_sms);
int launch_gram_mid(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                    cudaStream_t s, int64_t* launches);
/// The same Gram for M <= 8 rows (any K >= 1, incl. mode 0), one column per thread.
bool gram_small_supported(int64_t K, int64_t M, int64_t B);
int64_t gram_small_partials(int num_sms);
int launch_gram_small(const double* Y, int64_t K, int64_t M, int64_t B, double* partials, double* G, int num_sms,
                      cudaStream_t s, int64_t* launches);

/// Fused two-leaf reconstruction X = (U0 (x) U1) W per slab (k_decode.cu).
struct Decode2Args {
    const double* W;  // [r0][r1][T]
    int64_t T;
    int r0, r1;
    int64_t n0, n1;
    const double* U0;  // n0 x r0, column-major
    const double* U1;  // n1 x r1
    double* X;         // [n0][n1][T]
    const double* Y = nullptr;  // set: no X; one sum (X - Y)^2 per warp into partials
    double* partials = nullptr;
    // residual mode, optional: the last CTA sums the partials (fixed order)
    // into final_out[0] and, when given, final_host[0] (mapped host memory)
    double* final_out = nullptr;
    double* final_host = nullptr;
    unsigned int* ticket = nullptr;  // zero on entry, left zero on exit
};
bool decode2_supported(int64_t n0, int64_t n1, int64_t r0, int64_t r1);
int launch_decode2(const Decode2Args& a, int num_sms, cudaStream_t s, int64_t* launches);
/// Partials written by a residual-mode launch_decode2 over T slabs.
int64_t decode2_partials(int64_t T, int num_sms);
/// One sum (x - y)^2 per block into partials; returns the block count.
int launch_diff_sumsq(const double* x, const double* y, int64_t n, double* partials, int num_sms, cudaStream_t s,
                      int64_t* launches);

bool quad_supported(int64_t extent, int64_t rank);
/// Returns the grid size (number of partials written), -1 for an unaligned X.
int launch_quad(const QuadArgs& a, bool finish, int num_sms, cudaStream_t s, int64_t* launches);
void launch_tail3(const Tail3Args& a, cudaStream_t s, int64_t* launches);

}  // namespace htr
