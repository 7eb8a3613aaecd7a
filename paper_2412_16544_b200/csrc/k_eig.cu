// One-CTA symmetric eigen-solver (parallel cyclic Jacobi) and the
// re-orthonormalisation used by basis expansion.
//
// The reference truncates with a thin SVD of each unfolding
// (Eigen::BDCSVD, truncated_svd.hpp:29-45). Here the same spectrum is taken
// from the Gram G = M M^T (lambda = sigma^2, eigenvectors = left singular
// vectors), which the streaming kernels produce in one pass over the batch;
// the n x n eigenproblem (n <= a few hundred) runs in a single CTA.
#include <algorithm>

#include "kernels.cuh"

namespace htr {
namespace {

constexpr int kJacobiThreads = 1024;

/// Round-robin tournament (circle method): after `round` rounds player 0
/// stays at position 0 and positions 1..m-1 have rotated right by `round`.
__device__ __forceinline__ int tour_pos(int i, int round, int m) {
    if (i == 0) return 0;
    int k = (i - 1 - round) % (m - 1);
    if (k < 0) k += m - 1;
    return 1 + k;
}
constexpr int64_t kSmemMaxN = 112;   // A and V in shared memory: 2 * 112^2 * 8 B = 196 KB
constexpr int64_t kSmemMaxNA = 160;  // A alone in shared memory (200 KB), V in global memory

/// Jacobi rotation for the pair (p, q), or (c, s) = (1, 0) when a_pq is
/// negligible: relative to the diagonal (|a_pq| <= 1e-15 sqrt(|a_pp a_qq|),
/// the classical test) or absolutely, below 2^-53 (= u) of the input's
/// trace. The Gram the solver receives already carries ~n u tr(G) of
/// rounding error and every rotation leaves ~u max|A| in the entries it
/// touches, so chasing smaller off-diagonal entries (rotations among
/// noise-level eigenvalues) only burns sweeps; without the absolute floor a
/// Gram with a noise-level tail never meets the relative test and runs all
/// 40 sweeps. (Tight-eps truncations re-measure the small eigenvalues through
/// a second, projected Gram, whose own trace sets its floor.)
__device__ __forceinline__ bool jacobi_rotation(double app, double aqq, double apq, double floor_abs, double* c_out,
                                                double* s_out) {
    if (!(fabs(apq) > floor_abs && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq)))) return false;
    const double tau = (aqq - app) / (2.0 * apq);
    double t;
    if (fabs(tau) > 1e150) t = 0.5 / tau;
    else t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
    const double c = 1.0 / sqrt(1.0 + t * t);
    *c_out = c;
    *s_out = t * c;
    return true;
}

__global__ void __launch_bounds__(kJacobiThreads) jacobi_kernel(const double* __restrict__ G, int n,
                                                                double* __restrict__ lambda,
                                                                double* __restrict__ Vout, double* gwork,
                                                                int a_smem, int v_smem) {
    extern __shared__ double smem[];
    __shared__ double cs[512], sn[512];
    __shared__ int prs[512], qrs[512];
    __shared__ int rotated;

    const int tid = threadIdx.x, nt = blockDim.x;
    // A in shared memory up to n = 160; V too up to n = 112, else in global
    // memory (touched only by this CTA: bar.sync orders its updates)
    double* A = a_smem ? smem : gwork;
    double* V = v_smem ? smem + static_cast<int64_t>(n) * n : gwork + static_cast<int64_t>(n) * n;
    const int64_t nn = static_cast<int64_t>(n) * n;
    for (int64_t i = tid; i < nn; i += nt) {
        const int64_t r = i % n, c = i / n;
        // symmetrise defensively: the Gram kernels are exact mirrors already
        A[i] = 0.5 * (G[r + n * c] + G[c + n * r]);
        V[i] = r == c ? 1.0 : 0.0;
    }
    const int m = n + (n & 1);
    __syncthreads();

    const int half = m / 2;
    __shared__ double tr_abs;
    if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += fabs(A[i + static_cast<int64_t>(n) * i]);
        tr_abs = t;
    }
    __syncthreads();
    const double floor_abs = 0x1p-53 * tr_abs;
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < m - 1; ++round) {
            // phase 1: rotations for the disjoint pairs of this round
            for (int i = tid; i < half; i += nt) {
                int p = tour_pos(i, round, m), q = tour_pos(m - 1 - i, round, m);
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, s = 0.0;
                if (q < n &&
                    jacobi_rotation(A[p + static_cast<int64_t>(n) * p], A[q + static_cast<int64_t>(n) * q],
                                    A[p + static_cast<int64_t>(n) * q], floor_abs, &c, &s))
                    rotated = 1;
                cs[i] = c; sn[i] = s; prs[i] = p; qrs[i] = q;
            }
            __syncthreads();
            // phase 2: 2x2 blocks (P, Q): A' = J_P^T A J_Q over rows {p_P, q_P},
            // columns {p_Q, q_Q} in one pass, and V's column pairs
            const int blocks = half * half;
            for (int b = tid; b < blocks; b += nt) {
                const int P = b % half, Q = b / half;
                const int pP = prs[P], qP = qrs[P], pQ = prs[Q], qQ = qrs[Q];
                const double cP = cs[P], sP = sn[P], cQ = cs[Q], sQ = sn[Q];
                if ((sP == 0.0 && sQ == 0.0) || (qP >= n && qQ >= n)) continue;
                if (qP >= n) {  // row pair padded: only the column rotation of row pP
                    double* r0 = A + pP;
                    const double x = r0[static_cast<int64_t>(n) * pQ], y = r0[static_cast<int64_t>(n) * qQ];
                    r0[static_cast<int64_t>(n) * pQ] = cQ * x - sQ * y;
                    r0[static_cast<int64_t>(n) * qQ] = sQ * x + cQ * y;
                    continue;
                }
                if (qQ >= n) {  // column pair padded: only the row rotation of column pQ
                    double* col = A + static_cast<int64_t>(n) * pQ;
                    const double x = col[pP], y = col[qP];
                    col[pP] = cP * x - sP * y;
                    col[qP] = sP * x + cP * y;
                    continue;
                }
                double* a_pp = A + pP + static_cast<int64_t>(n) * pQ;
                double* a_pq = A + pP + static_cast<int64_t>(n) * qQ;
                double* a_qp = A + qP + static_cast<int64_t>(n) * pQ;
                double* a_qq = A + qP + static_cast<int64_t>(n) * qQ;
                const double x00 = *a_pp, x01 = *a_pq, x10 = *a_qp, x11 = *a_qq;
                const double y00 = cP * x00 - sP * x10, y01 = cP * x01 - sP * x11;
                const double y10 = sP * x00 + cP * x10, y11 = sP * x01 + cP * x11;
                double z00 = cQ * y00 - sQ * y01, z01 = sQ * y00 + cQ * y01;
                double z10 = cQ * y10 - sQ * y11, z11 = sQ * y10 + cQ * y11;
                if (P == Q && sP != 0.0) { z01 = 0.0; z10 = 0.0; }  // annihilated pair
                *a_pp = z00; *a_pq = z01; *a_qp = z10; *a_qq = z11;
            }
            const int vitems = half * n;
            for (int it = tid; it < vitems; it += nt) {
                const int Q = it / n, r = it - Q * n;
                const double s = sn[Q];
                if (s == 0.0) continue;
                const double c = cs[Q];
                double* vp = V + static_cast<int64_t>(n) * prs[Q] + r;
                double* vq = V + static_cast<int64_t>(n) * qrs[Q] + r;
                const double x = *vp, y = *vq;
                *vp = c * x - s * y;
                *vq = s * x + c * y;
            }
            __syncthreads();
        }
        __syncthreads();
        if (!rotated) break;
        __syncthreads();
    }

    // sort eigenpairs by descending eigenvalue (stable on index)
    for (int i = tid; i < n; i += nt) {
        const double li = A[i + static_cast<int64_t>(n) * i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double lj = A[j + static_cast<int64_t>(n) * j];
            rank += (lj > li) || (lj == li && j < i);
        }
        lambda[rank] = li;
        for (int r = 0; r < n; ++r) Vout[r + static_cast<int64_t>(n) * rank] = V[r + static_cast<int64_t>(n) * i];
    }
}

// --------------------------------------------------------------------------
// n <= kSymMaxN: the same rounds with A stored as its packed lower triangle,
// so that A and V both fit in shared memory up to n = 135 (c5's 128-row leaf
// Grams, whose V previously lived in global memory), and only the 2x2 blocks
// P <= Q are updated (A' = J^T A J stays exactly symmetric; the (Q, P) block
// is the transpose held in the same entries).
// --------------------------------------------------------------------------
constexpr int kSymMaxN = 184;        // with V split over CTAs (below)
constexpr int kSymOneCta = 135;      // n(n+1)/2 + n^2 doubles = 194 KB at n = 135
constexpr int kSymSmemDoubles = 27136;  // dynamic shared memory budget (212 KB)
constexpr int kEigBatchMax = 16;     // CTAs per launch

/// CTAs over which a solve's V rows are split: each CTA carries the whole
/// packed A (it evolves identically in every CTA: same inputs, same code)
/// and the rows [r0, r1) of V, so that A plus its V share fits in shared
/// memory (n = 144, c3's transfer residual: 2 CTAs).
__host__ __device__ __forceinline__ int sym_splits(int n) {
    const int np = n * (n + 1) / 2;
    for (int k = 1; k <= 4; ++k)
        if (np + ((n + k - 1) / k) * n <= kSymSmemDoubles) return k;
    return 0;
}

__device__ __forceinline__ int sym_idx(int i, int j, int n) {  // packed lower, column-major
    if (i < j) { const int t = i; i = j; j = t; }
    return j * n - ((j * (j + 1)) >> 1) + i;
}

// one CTA per job of the batch: independent eigenproblems (the leaf Grams of
// one layer) run side by side; each CTA's arithmetic does not depend on the
// batch or the block size, so a batched solve equals the single ones bit for bit
struct SymJobs {
    const double* G[kEigBatchMax];
    double* lambda[kEigBatchMax];  // null on the CTAs that do not write eigenvalues
    double* V[kEigBatchMax];
    int n[kEigBatchMax];
    int r0[kEigBatchMax], r1[kEigBatchMax];  // V rows held by this CTA
};

__global__ void __launch_bounds__(kJacobiThreads) jacobi_sym_kernel(const SymJobs jobs) {
    const double* __restrict__ G = jobs.G[blockIdx.x];
    const int n = jobs.n[blockIdx.x];
    double* __restrict__ lambda = jobs.lambda[blockIdx.x];
    double* __restrict__ Vout = jobs.V[blockIdx.x];
    const int vr0 = jobs.r0[blockIdx.x], nr = jobs.r1[blockIdx.x] - vr0;
    extern __shared__ double smem[];
    // rotation parameters, double-buffered by round parity: round r + 1's are
    // computed while round r's V column pairs are being rotated
    __shared__ double cs2[2][kSymMaxN / 2 + 1], sn2[2][kSymMaxN / 2 + 1];
    __shared__ int prs2[2][kSymMaxN / 2 + 1], qrs2[2][kSymMaxN / 2 + 1];
    __shared__ int rotated;
    __shared__ double tr_abs;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int np = (n * (n + 1)) / 2;
    double* A = smem;       // packed lower triangle
    double* V = smem + np;  // rows [vr0, vr0 + nr) of V (nr x n, column-major)
    for (int j = 0; j < n; ++j)
        for (int i = j + tid; i < n; i += nt)
            A[sym_idx(i, j, n)] = 0.5 * (G[i + static_cast<int64_t>(n) * j] + G[j + static_cast<int64_t>(n) * i]);
    for (int e = tid; e < nr * n; e += nt) V[e] = (vr0 + e % nr == e / nr) ? 1.0 : 0.0;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += fabs(A[sym_idx(i, i, n)]);
        tr_abs = t;
    }
    __syncthreads();
    const double floor_abs = 0x1p-53 * tr_abs;
    const int m = n + (n & 1), half = m / 2;
    const int vq0 = tid / nr, vrr0 = tid - vq0 * nr, vqs = nt / nr, vrs = nt - vqs * nr;
    auto rotations = [&](int round, int buf) {
        for (int i = tid; i < half; i += nt) {
            int p = tour_pos(i, round, m), q = tour_pos(m - 1 - i, round, m);
            if (p > q) { const int t = p; p = q; q = t; }
            double c = 1.0, s = 0.0;
            if (q < n && jacobi_rotation(A[sym_idx(p, p, n)], A[sym_idx(q, q, n)], A[sym_idx(p, q, n)], floor_abs,
                                         &c, &s))
                rotated = 1;
            cs2[buf][i] = c; sn2[buf][i] = s; prs2[buf][i] = p; qrs2[buf][i] = q;
        }
    };
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        rotations(0, 0);
        __syncthreads();
        for (int round = 0; round < m - 1; ++round) {
            const int buf = round & 1;
            const double* cs = cs2[buf];
            const double* sn = sn2[buf];
            const int* prs = prs2[buf];
            const int* qrs = qrs2[buf];
            // blocks P <= Q: warp w takes the column pairs Q = qq and
            // Q' = half - 1 - qq together (qq + 1 and Q' + 1 blocks: half + 1
            // per qq) and its lanes stride over the concatenated P ranges
            const int lane = tid & 31, nwarps = nt >> 5;
            for (int qq = tid >> 5; qq <= half - 1 - qq; qq += nwarps) {
              const int q2 = half - 1 - qq;
              const int cnt = qq == q2 ? qq + 1 : half + 1;
              for (int e = lane; e < cnt; e += 32) {
                const int Q = e <= qq ? qq : q2;
                const int P = e <= qq ? e : e - qq - 1;
                const double cP = cs[P], sP = sn[P], cQ = cs[Q], sQ = sn[Q];
                if (sP == 0.0 && sQ == 0.0) continue;
                const int pP = prs[P], qP = qrs[P], pQ = prs[Q], qQ = qrs[Q];
                const bool okr = qP < n, okc = qQ < n;
                if (P == Q) {
                    if (!okr) continue;
                    // diagonal block: [a_pp a_pq; a_pq a_qq] -> diag(.), pair annihilated
                    const int ipp = sym_idx(pP, pP, n), iqq = sym_idx(qP, qP, n), ipq = sym_idx(pP, qP, n);
                    const double x00 = A[ipp], x01 = A[ipq], x11 = A[iqq];
                    const double y00 = cP * x00 - sP * x01, y01 = cP * x01 - sP * x11;
                    const double y10 = sP * x00 + cP * x01, y11 = sP * x01 + cP * x11;
                    A[ipp] = cP * y00 - sP * y01;
                    A[iqq] = sP * y10 + cP * y11;
                    A[ipq] = 0.0;
                    continue;
                }
                const int i00 = sym_idx(pP, pQ, n);
                const int i01 = okc ? sym_idx(pP, qQ, n) : 0;
                const int i10 = okr ? sym_idx(qP, pQ, n) : 0;
                const int i11 = (okr && okc) ? sym_idx(qP, qQ, n) : 0;
                const double x00 = A[i00], x01 = okc ? A[i01] : 0.0, x10 = okr ? A[i10] : 0.0,
                             x11 = (okr && okc) ? A[i11] : 0.0;
                const double y00 = cP * x00 - sP * x10, y01 = cP * x01 - sP * x11;
                const double y10 = sP * x00 + cP * x10, y11 = sP * x01 + cP * x11;
                A[i00] = cQ * y00 - sQ * y01;
                if (okc) A[i01] = sQ * y00 + cQ * y01;
                if (okr) A[i10] = cQ * y10 - sQ * y11;
                if (okr && okc) A[i11] = sQ * y10 + cQ * y11;
              }
            }
            __syncthreads();  // A after this round: the next round's rotations
            if (round + 1 < m - 1) rotations(round + 1, buf ^ 1);
            // V's column pairs: (Q, r) items walked incrementally (no division)
            for (int Q = vq0, r = vrr0; Q < half; Q += vqs, r += vrs) {
                if (r >= nr) {
                    r -= nr;
                    ++Q;
                    if (Q >= half) break;
                }
                const double s = sn[Q];
                if (s == 0.0) continue;
                const double c = cs[Q];
                double* vp = V + nr * prs[Q] + r;
                double* vq = V + nr * qrs[Q] + r;
                const double x = *vp, y = *vq;
                *vp = c * x - s * y;
                *vq = s * x + c * y;
            }
            __syncthreads();
        }
        __syncthreads();
        if (!rotated) break;
        __syncthreads();
    }
    // sort eigenpairs by descending eigenvalue (stable on index)
    for (int i = tid; i < n; i += nt) {
        const double li = A[sym_idx(i, i, n)];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double lj = A[sym_idx(j, j, n)];
            rank += (lj > li) || (lj == li && j < i);
        }
        if (lambda) lambda[rank] = li;
        for (int r = 0; r < nr; ++r) Vout[vr0 + r + static_cast<int64_t>(n) * rank] = V[r + nr * i];
    }
}

// --------------------------------------------------------------------------
// Large n: the same parallel cyclic Jacobi spread over a cluster of CTAs.
// A and V live in global memory (L2); every CTA computes the round's
// rotations itself (bit-identical: same inputs, same code), applies its
// share of the 2x2 blocks A[{p,q}_P, {p,q}_Q] <- J_P^T A J_Q and of V's
// column pairs in ONE pass, and the round ends with a single cluster
// barrier (release/acquire orders the global-memory updates).
// --------------------------------------------------------------------------
constexpr int kClusterCTAs = 8;
constexpr int kClusterThreads = 512;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__global__ void __cluster_dims__(kClusterCTAs, 1, 1) __launch_bounds__(kClusterThreads)
    jacobi_cluster_kernel(const double* __restrict__ G, int n, double* __restrict__ lambda, double* __restrict__ Vout,
                          double* A, double* V) {
    __shared__ double cs[kJacobiMaxN / 2], sn[kJacobiMaxN / 2];
    __shared__ int prs[kJacobiMaxN / 2], qrs[kJacobiMaxN / 2];
    __shared__ int rotated;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int crank = static_cast<int>(cluster_rank());
    const int gtid = crank * nt + tid, gnt = kClusterCTAs * nt;
    const int64_t nn = static_cast<int64_t>(n) * n;
    for (int64_t i = gtid; i < nn; i += gnt) {
        const int64_t r = i % n, c = i / n;
        A[i] = 0.5 * (G[r + n * c] + G[c + n * r]);
        V[i] = r == c ? 1.0 : 0.0;
    }
    const int m = n + (n & 1);
    const int half = m / 2;
    cluster_sync_all();
    __shared__ double tr_abs;
    if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += fabs(A[i + static_cast<int64_t>(n) * i]);
        tr_abs = t;  // identical in every CTA (same inputs, same order)
    }
    __syncthreads();
    const double floor_abs = 0x1p-53 * tr_abs;

    for (int sweep = 0; sweep < 40; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int round = 0; round < m - 1; ++round) {
            for (int i = tid; i < half; i += nt) {
                int p = tour_pos(i, round, m), q = tour_pos(m - 1 - i, round, m);
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, s = 0.0;
                if (q < n &&
                    jacobi_rotation(A[p + static_cast<int64_t>(n) * p], A[q + static_cast<int64_t>(n) * q],
                                    A[p + static_cast<int64_t>(n) * q], floor_abs, &c, &s))
                    rotated = 1;
                cs[i] = c; sn[i] = s; prs[i] = p; qrs[i] = q;
            }
            __syncthreads();
            // every CTA finished reading A for the rotations before anyone writes
            cluster_sync_all();
            // 2x2 blocks (P, Q): A' = J_P^T A J_Q over rows {p_P, q_P}, cols
            // {p_Q, q_Q}, then V's column pairs. Items are disjoint, so each
            // thread issues the loads of kBatch items before any store (A and
            // V are in L2: one round trip per batch instead of per item). A
            // padded pair (q = n, odd n) has s = 0, so its rotation is the
            // identity and only its in-range entries are touched.
            constexpr int kBatch = 2;
            const int blocks = half * half;
            for (int b0 = gtid; b0 < blocks; b0 += kBatch * gnt) {
                double x[kBatch][4];
                int off[kBatch][4];  // n <= 2048: n^2 fits 32 bits
                bool live[kBatch], okr[kBatch], okc[kBatch];
                double c_p[kBatch], s_p[kBatch], c_q[kBatch], s_q[kBatch];
                bool diag[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int b = b0 + u * gnt;
                    live[u] = false;
                    if (b >= blocks) continue;
                    const int P = b / half, Q = b - P * half;
                    c_p[u] = cs[P]; s_p[u] = sn[P]; c_q[u] = cs[Q]; s_q[u] = sn[Q];
                    if (s_p[u] == 0.0 && s_q[u] == 0.0) continue;
                    const int pP = prs[P], qP = qrs[P], pQ = prs[Q], qQ = qrs[Q];
                    okr[u] = qP < n;
                    okc[u] = qQ < n;
                    diag[u] = P == Q;
                    live[u] = true;
                    off[u][0] = pP + n * pQ;
                    off[u][1] = pP + n * qQ;
                    off[u][2] = qP + n * pQ;
                    off[u][3] = qP + n * qQ;
                    x[u][0] = A[off[u][0]];
                    x[u][1] = okc[u] ? A[off[u][1]] : 0.0;
                    x[u][2] = okr[u] ? A[off[u][2]] : 0.0;
                    x[u][3] = (okr[u] && okc[u]) ? A[off[u][3]] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (!live[u]) continue;
                    const double cP = c_p[u], sP = s_p[u], cQ = c_q[u], sQ = s_q[u];
                    const double y00 = cP * x[u][0] - sP * x[u][2], y01 = cP * x[u][1] - sP * x[u][3];
                    const double y10 = sP * x[u][0] + cP * x[u][2], y11 = sP * x[u][1] + cP * x[u][3];
                    double z00 = cQ * y00 - sQ * y01, z01 = sQ * y00 + cQ * y01;
                    double z10 = cQ * y10 - sQ * y11, z11 = sQ * y10 + cQ * y11;
                    if (diag[u] && sP != 0.0) { z01 = 0.0; z10 = 0.0; }  // annihilated pair
                    A[off[u][0]] = z00;
                    if (okc[u]) A[off[u][1]] = z01;
                    if (okr[u]) A[off[u][2]] = z10;
                    if (okr[u] && okc[u]) A[off[u][3]] = z11;
                }
            }
            // V <- V J (column pairs), batched the same way
            const int vitems = half * n;
            for (int i0 = gtid; i0 < vitems; i0 += kBatch * gnt) {
                double vx[kBatch], vy[kBatch], vc[kBatch], vs[kBatch];
                int vpp[kBatch], vqq[kBatch];
                bool vl[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int it = i0 + u * gnt;
                    vl[u] = false;
                    if (it >= vitems) continue;
                    const int Q = it / n, r = it - Q * n;
                    vs[u] = sn[Q];
                    if (vs[u] == 0.0) continue;
                    vc[u] = cs[Q];
                    vpp[u] = n * prs[Q] + r;
                    vqq[u] = n * qrs[Q] + r;
                    vx[u] = V[vpp[u]];
                    vy[u] = V[vqq[u]];
                    vl[u] = true;
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (!vl[u]) continue;
                    V[vpp[u]] = vc[u] * vx[u] - vs[u] * vy[u];
                    V[vqq[u]] = vs[u] * vx[u] + vc[u] * vy[u];
                }
            }
            cluster_sync_all();
        }
        __syncthreads();
        if (!rotated) break;  // identical decision in every CTA
        __syncthreads();
    }
    // sort eigenpairs by descending eigenvalue (stable on index)
    for (int i = gtid; i < n; i += gnt) {
        const double li = A[i + static_cast<int64_t>(n) * i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double lj = A[j + static_cast<int64_t>(n) * j];
            rank += (lj > li) || (lj == li && j < i);
        }
        lambda[rank] = li;
        for (int r = 0; r < n; ++r) Vout[r + static_cast<int64_t>(n) * rank] = V[r + static_cast<int64_t>(n) * i];
    }
}

// --------------------------------------------------------------------------
// Positive-definiteness test of G - shift I (full-rank truncations): a
// right-looking Cholesky in one CTA; flag[0] = 1 if every pivot is positive.
// Cholesky is backward stable, so success certifies lambda_min(G) > shift up
// to ~n u ||G||, which the caller's margin covers.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) posdef_kernel(const double* __restrict__ G, int n, double shift,
                                                      double* __restrict__ A, double* __restrict__ flag) {
    __shared__ double colk[kJacobiMaxN];
    __shared__ int ok;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t nn = static_cast<int64_t>(n) * n;
    for (int64_t e = tid; e < nn; e += nt) {
        const int64_t r = e % n, c = e / n;
        A[e] = (r >= c) ? G[e] - (r == c ? shift : 0.0) : 0.0;  // lower triangle
    }
    if (tid == 0) ok = 1;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        const double piv = A[k + static_cast<int64_t>(n) * k];
        if (!(piv > 0.0)) {  // uniform: every thread reads the same pivot
            if (tid == 0) ok = 0;
            break;
        }
        const double inv = 1.0 / sqrt(piv);
        const int m = n - k - 1;
        for (int i = tid; i < m; i += nt) {
            const double v = A[(k + 1 + i) + static_cast<int64_t>(n) * k] * inv;
            A[(k + 1 + i) + static_cast<int64_t>(n) * k] = v;
            colk[i] = v;
        }
        __syncthreads();
        // trailing lower triangle: A[i, j] -= l_i l_j for k < j <= i; warp w
        // takes columns j = w, w + 32, ..., its lanes run down the column
        const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
        for (int j = warp; j < m; j += nw) {
            const double lj = colk[j];
            double* col = A + static_cast<int64_t>(n) * (k + 1 + j) + (k + 1);
            for (int i = j + lane; i < m; i += 32) col[i] -= colk[i] * lj;
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0) flag[0] = ok ? 1.0 : 0.0;
}

// --------------------------------------------------------------------------
// Blocked form of the same test (panels of 32 columns; the runtime runs the
// trailing updates A22 -= P P^T on the DMMA GEMM engine between panels).
// --------------------------------------------------------------------------
constexpr int kCholB = 32;

__global__ void chol_prepare_kernel(const double* __restrict__ G, int n, double shift, double* __restrict__ A,
                                    double* __restrict__ flag) {
    const int64_t nn = static_cast<int64_t>(n) * n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nn;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % n, c = e / n;
        A[e] = G[e] - (r == c ? shift : 0.0);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) flag[0] = 1.0;
}

/// Columns [kb, kb + b) of rows [kb, n): the b x b diagonal block by one
/// warp (lane i owns row i; no block barrier per column), the rows below by
/// forward substitution against it, one row per thread (b = 32 there: only
/// the last panel is narrower, and it has no rows below). A non-positive
/// pivot clears flag[0]; later panels then return at once.
__global__ void __launch_bounds__(256, 1) chol_panel_kernel(double* __restrict__ A, int n, int kb, int b,
                                                         double* __restrict__ flag) {
    __shared__ double D[kCholB][kCholB + 1];
    __shared__ int ok;
    if (flag[0] != 1.0) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < b * b; e += nt) {
        const int i = e % b, j = e / b;
        D[i][j] = i >= j ? A[(kb + i) + static_cast<int64_t>(n) * (kb + j)] : 0.0;
    }
    if (tid == 0) ok = 1;
    __syncthreads();
    if (tid < 32) {
        const int lane = tid;
        for (int k = 0; k < b; ++k) {
            const double piv = D[k][k];
            if (!(piv > 0.0)) {  // the same value in every lane
                if (lane == 0) ok = 0;
                break;
            }
            const double lkk = sqrt(piv);
            __syncwarp();
            if (lane == k) D[k][k] = lkk;
            if (lane > k && lane < b) D[lane][k] /= lkk;
            __syncwarp();
            if (lane > k && lane < b) {
                const double lik = D[lane][k];
                for (int j = k + 1; j <= lane; ++j) D[lane][j] -= lik * D[j][k];
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (!ok) {
        if (tid == 0) flag[0] = 0.0;
        return;
    }
    for (int e = tid; e < b * b; e += nt) {
        const int i = e % b, j = e / b;
        if (i >= j) A[(kb + i) + static_cast<int64_t>(n) * (kb + j)] = D[i][j];
    }
    if (b != kCholB) return;
    // (volatile: the factor is re-read from shared memory per row instead of
    // being hoisted into 528 registers)
    volatile double(*Dv)[kCholB + 1] = D;
    __shared__ double Dinv[kCholB];
    if (tid < kCholB) Dinv[tid] = 1.0 / D[tid][tid];
    __syncthreads();
    volatile double* Di = Dinv;
    for (int r = kb + kCholB + tid; r < n; r += nt) {
        double x[kCholB];
#pragma unroll
        for (int j = 0; j < kCholB; ++j) x[j] = A[r + static_cast<int64_t>(n) * (kb + j)];
#pragma unroll
        for (int j = 0; j < kCholB; ++j) {
            double v = x[j];
#pragma unroll
            for (int l = 0; l < j; ++l) v = fma(-Dv[j][l], x[l], v);
            x[j] = v * Di[j];
        }
#pragma unroll
        for (int j = 0; j < kCholB; ++j) A[r + static_cast<int64_t>(n) * (kb + j)] = x[j];
    }
}

// --------------------------------------------------------------------------
// Re-orthonormalisation of new directions (expand_core, ht_rise.hpp:53-79):
// W <- (I - U U^T) W twice, then CholeskyQR2. One CTA; all sizes small.
// --------------------------------------------------------------------------
__device__ void block_project_out(const double* U, int64_t alpha, int64_t r, double* W, int64_t q, double* T) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t ab = tid; ab < r * q; ab += nt) {
        const int64_t a = ab % r, b = ab / r;
        double s = 0.0;
        for (int64_t i = 0; i < alpha; ++i) s = fma(U[i + alpha * a], W[i + alpha * b], s);
        T[ab] = s;
    }
    __syncthreads();
    for (int64_t ib = tid; ib < alpha * q; ib += nt) {
        const int64_t i = ib % alpha, b = ib / alpha;
        double s = 0.0;
        for (int64_t a = 0; a < r; ++a) s = fma(U[i + alpha * a], T[a + r * b], s);
        W[ib] -= s;
    }
    __syncthreads();
}

__device__ void block_cholqr(int64_t alpha, double* W, int64_t q, double* Gm) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t ab = tid; ab < q * q; ab += nt) {
        const int64_t a = ab % q, b = ab / q;
        double s = 0.0;
        for (int64_t i = 0; i < alpha; ++i) s = fma(W[i + alpha * a], W[i + alpha * b], s);
        Gm[ab] = s;
    }
    __syncthreads();
    // in-place lower Cholesky G = L L^T (right-looking)
    for (int64_t k = 0; k < q; ++k) {
        if (tid == 0) Gm[k + q * k] = sqrt(fmax(Gm[k + q * k], 1e-300));
        __syncthreads();
        const double dkk = Gm[k + q * k];
        for (int64_t i = k + 1 + tid; i < q; i += nt) Gm[i + q * k] /= dkk;
        __syncthreads();
        const int64_t rem = q - k - 1;
        for (int64_t ij = tid; ij < rem * rem; ij += nt) {
            const int64_t i = k + 1 + ij % rem, j = k + 1 + ij / rem;
            if (j <= i) Gm[i + q * j] -= Gm[i + q * k] * Gm[j + q * k];
        }
        __syncthreads();
    }
    // W <- W L^{-T}: each row w solves L x = w^T (forward substitution)
    for (int64_t i = tid; i < alpha; i += nt) {
        for (int64_t j = 0; j < q; ++j) {
            double s = W[i + alpha * j];
            for (int64_t k = 0; k < j; ++k) s -= Gm[j + q * k] * W[i + alpha * k];
            W[i + alpha * j] = s / Gm[j + q * j];
        }
    }
    __syncthreads();
}

/// CholeskyQR2 of W (alpha x q, q <= 32) staged in shared memory: the Gram
/// by warps (lanes over rows, shuffle sums), its Cholesky by one warp (lane
/// = row, no block barrier per column), W L^{-T} by forward substitution
/// one row per thread. The polish of every truncation's retained basis.
constexpr int kQrMaxQ = 32;
__global__ void __launch_bounds__(512) cholqr2_smem_kernel(double* __restrict__ Wg, int alpha, int q,
                                                           double* __restrict__ info) {
    extern __shared__ double Ws[];  // alpha x q, column-major
    __shared__ double L[kQrMaxQ][kQrMaxQ + 1];
    __shared__ double Linv[kQrMaxQ];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int n = alpha * q;
    for (int e = tid; e < n; e += nt) Ws[e] = Wg[e];
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
        for (int ab = warp; ab < q * q; ab += nw) {
            const int a = ab % q, b = ab / q;
            if (a < b) continue;
            const double* wa = Ws + alpha * a;
            const double* wb = Ws + alpha * b;
            double s = 0.0;
            for (int i = lane; i < alpha; i += 32) s = fma(wa[i], wb[i], s);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) L[a][b] = s;
        }
        __syncthreads();
        if (warp == 0) {  // in-place lower Cholesky, lane = row
            for (int k = 0; k < q; ++k) {
                const double dkk = sqrt(fmax(L[k][k], 1e-300));
                __syncwarp();
                if (lane == k) { L[k][k] = dkk; Linv[k] = 1.0 / dkk; }
                if (lane > k && lane < q) L[lane][k] /= dkk;
                __syncwarp();
                if (lane > k && lane < q) {
                    const double lik = L[lane][k];
                    for (int j = k + 1; j <= lane; ++j) L[lane][j] -= lik * L[j][k];
                }
                __syncwarp();
            }
        }
        __syncthreads();
        for (int i = tid; i < alpha; i += nt)
            for (int j = 0; j < q; ++j) {
                double v = Ws[i + alpha * j];
                for (int k = 0; k < j; ++k) v = fma(-L[j][k], Ws[i + alpha * k], v);
                Ws[i + alpha * j] = v * Linv[j];
            }
        __syncthreads();
    }
    for (int e = tid; e < n; e += nt) Wg[e] = Ws[e];
    if (tid == 0 && info) {  // no old basis: defect 0, ||W||_F of an orthonormal W
        info[0] = 0.0;
        info[1] = sqrt(static_cast<double>(q));
    }
}

__global__ void __launch_bounds__(512) orthonormalize_kernel(const double* U, int64_t alpha, int64_t r, double* W,
                                                             int64_t q, double* info, double* work) {
    double* T = work;                 // r * q
    double* Gm = work + r * q;        // q * q
    if (r > 0) {
        block_project_out(U, alpha, r, W, q, T);
        block_project_out(U, alpha, r, W, q, T);
    }
    block_cholqr(alpha, W, q, Gm);
    block_cholqr(alpha, W, q, Gm);
    // defect ||U^T W||_F and ||W||_F (expand_core's orthogonality check)
    __shared__ double red[2][16];
    double d = 0.0, w = 0.0;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t ab = tid; ab < r * q; ab += nt) {
        const int64_t a = ab % r, b = ab / r;
        double s = 0.0;
        for (int64_t i = 0; i < alpha; ++i) s = fma(U[i + alpha * a], W[i + alpha * b], s);
        d = fma(s, s, d);
    }
    for (int64_t i = tid; i < alpha * q; i += nt) w = fma(W[i], W[i], w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        w += __shfl_xor_sync(0xffffffffu, w, o);
    }
    if ((tid & 31) == 0) { red[0][tid >> 5] = d; red[1][tid >> 5] = w; }
    __syncthreads();
    if (tid == 0) {
        double sd = 0.0, sw = 0.0;
        for (int k = 0; k < nt / 32; ++k) { sd += red[0][k]; sw += red[1][k]; }
        info[0] = sqrt(sd);
        info[1] = sqrt(sw);
    }
}

}  // namespace

void launch_jacobi_eig(const double* G, int64_t n, double* lambda, double* V, double* work, cudaStream_t s,
                       int64_t* launches) {
    if (jacobi_batchable(n)) {
        launch_jacobi_eig_batch(&G, &n, &lambda, &V, 1, s, launches);
        return;
    }
    if (n > kSmemMaxNA) {
        jacobi_cluster_kernel<<<kClusterCTAs, kClusterThreads, 0, s>>>(G, static_cast<int>(n), lambda, V, work,
                                                                       work + n * n);
        ++*launches;
        return;
    }
    const bool v_smem = n <= kSmemMaxN;
    const size_t smem = (v_smem ? 2 : 1) * sizeof(double) * static_cast<size_t>(n * n);
    // static + dynamic shared memory above 48 KB needs the opt-in (the
    // kernel's static arrays take ~17 KB): raise the limit once to the
    // largest in-smem problem
    ensure_smem_limit(reinterpret_cast<const void*>(jacobi_kernel),
                      sizeof(double) * std::max(2 * kSmemMaxN * kSmemMaxN, kSmemMaxNA * kSmemMaxNA));
    const int threads = n <= 32 ? 128 : (n <= 64 ? 256 : kJacobiThreads);
    jacobi_kernel<<<1, threads, smem, s>>>(G, static_cast<int>(n), lambda, V, work, 1, v_smem ? 1 : 0);
    ++*launches;
}

bool jacobi_batchable(int64_t n) { return n >= 1 && n <= kSymMaxN && sym_splits(static_cast<int>(n)) > 0; }

void launch_jacobi_eig_batch(const double* const* G, const int64_t* n, double* const* lambda, double* const* V,
                             int count, cudaStream_t s, int64_t* launches) {
    ensure_smem_limit(reinterpret_cast<const void*>(jacobi_sym_kernel), sizeof(double) * kSymSmemDoubles);
    SymJobs jobs{};
    int blocks = 0;
    int64_t smem_max = 0, nmax = 0;
    auto flush = [&] {
        if (blocks == 0) return;
        const int threads = nmax <= 32 ? 128 : (nmax <= 64 ? 256 : kJacobiThreads);
        jacobi_sym_kernel<<<blocks, threads, sizeof(double) * static_cast<size_t>(smem_max), s>>>(jobs);
        ++*launches;
        jobs = SymJobs{};
        blocks = 0;
        smem_max = nmax = 0;
    };
    for (int i = 0; i < count; ++i) {
        const int ni = static_cast<int>(n[i]);
        const int k = sym_splits(ni);
        if (blocks + k > kEigBatchMax) flush();
        const int rows = (ni + k - 1) / k;
        for (int j = 0; j < k; ++j) {
            jobs.G[blocks] = G[i];
            jobs.lambda[blocks] = j == 0 ? lambda[i] : nullptr;
            jobs.V[blocks] = V[i];
            jobs.n[blocks] = ni;
            jobs.r0[blocks] = std::min(ni, j * rows);
            jobs.r1[blocks] = std::min(ni, (j + 1) * rows);
            ++blocks;
        }
        smem_max = std::max<int64_t>(smem_max, ni * (ni + 1) / 2 + static_cast<int64_t>(rows) * ni);
        nmax = std::max<int64_t>(nmax, ni);
    }
    flush();
}

void launch_posdef_test(const double* G, int64_t n, double shift, double* work, double* flag, cudaStream_t s,
                        int64_t* launches) {
    posdef_kernel<<<1, 1024, 0, s>>>(G, static_cast<int>(n), shift, work, flag);
    ++*launches;
}

void launch_chol_prepare(const double* G, int64_t n, double shift, double* A, double* flag, cudaStream_t s,
                         int64_t* launches) {
    const int64_t nn = n * n;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(296, (nn + 255) / 256)));
    chol_prepare_kernel<<<blocks, 256, 0, s>>>(G, static_cast<int>(n), shift, A, flag);
    ++*launches;
}

void launch_chol_panel(double* A, int64_t n, int64_t kb, int64_t b, double* flag, cudaStream_t s, int64_t* launches) {
    chol_panel_kernel<<<1, 256, 0, s>>>(A, static_cast<int>(n), static_cast<int>(kb), static_cast<int>(b), flag);
    ++*launches;
}

void launch_orthonormalize_new(const double* U, int64_t alpha, int64_t r, double* W, int64_t q, double* info,
                               double* work, cudaStream_t s, int64_t* launches) {
    if (r == 0 && q >= 1 && q <= kQrMaxQ && alpha * q <= 16384) {
        // the polish of a fresh basis (no old columns): shared-memory CholeskyQR2
        const size_t smem = sizeof(double) * static_cast<size_t>(alpha * q);
        ensure_smem_limit(reinterpret_cast<const void*>(cholqr2_smem_kernel), smem);
        cholqr2_smem_kernel<<<1, 512, smem, s>>>(W, static_cast<int>(alpha), static_cast<int>(q), info);
        ++*launches;
        return;
    }
    orthonormalize_kernel<<<1, 512, 0, s>>>(U, alpha, r, W, q, info, work);
    ++*launches;
}

}  // namespace htr
