// htrise-b200 native runtime: device memory, representations, algorithms.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "htrise/dimension_tree.hpp"
#include "htrise_cuda.h"
#include "kernels.cuh"

namespace htr {

using htrise::DimensionTree;
using htrise::Index;
using htrise::NodeId;
using htrise::NodeKind;
using htrise::RankMap;
using htrise::Shape;
using htrise::TreeNode;

struct Error {
    htr_status code;
    std::string msg;
};
[[noreturn]] void raise(htr_status code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, int line);
#define HTR_CUDA(x) ::htr::cuda_check((x), #x, __LINE__)

/// Owns the context's CUDA stream; shared by every buffer allocated on it so
/// stream-ordered frees stay valid after the context handle is destroyed.
struct Stream {
    cudaStream_t s = nullptr;
    int device = 0;
    explicit Stream(int dev);
    ~Stream();
    // Host-side free lists of stream-ordered blocks (power-of-two size
    // classes up to 256 MB, at most 1 GB held): a block released by one Buf is handed to the next
    // allocation of its class without a driver call. All work is enqueued on
    // `s`, so the hand-over has exactly cudaFreeAsync + cudaMallocAsync's
    // ordering on that stream; it saves their ~2 us of host time per buffer,
    // which the latency-bound skip updates (configs 2, 3) pay 5-6 times a batch,
    // and the ~0.4 ms a 100 MB cudaMallocAsync can take (config 5's BHT-l2r
    // waited that long for its projected tensor).
    static constexpr int kMinClass = 5, kMaxClass = 25;  // 2^5 .. 2^25 doubles
    static constexpr size_t kCacheCapBytes = size_t{1024} << 20;
    std::mutex mu;
    std::vector<double*> bins[kMaxClass + 1];
    size_t cached_bytes = 0;
    /// Size class of n doubles, or -1 when the block is not cached.
    static int size_class(int64_t n);
    double* take(int cls);
    bool give(int cls, double* p);
};
using StreamPtr = std::shared_ptr<Stream>;

/// Stream-ordered device allocation of n doubles.
struct Buf {
    StreamPtr st;
    double* p = nullptr;
    int64_t n = 0;
    bool owned = true;
    bool identity = false;  // holds exactly the identity matrix (a full-rank node's basis)
    Buf(StreamPtr st_, int64_t n_);
    /// Non-owning wrapper around caller memory (device pointers handed in
    /// through the C-ABI).
    Buf(StreamPtr st_, double* external, int64_t n_) : st(std::move(st_)), p(external), n(n_), owned(false) {}
    int cls = -1;  // size class of a cached block (Stream::size_class)
    ~Buf();
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
};
using BufPtr = std::shared_ptr<Buf>;

/// Device tensor view: canonical layout, shared immutable storage.
struct DT {
    BufPtr buf;
    Shape shape;
    int64_t offset = 0;
    double* data() const { return buf->p + offset; }
    int64_t size() const { return htrise::shape_product(shape); }
};

/// Append-only root core r11 x r12 x capacity (batch axis last). Several
/// representation values may share it; each sees its first `acc` slices.
struct RootStore {
    BufPtr buf;
    int64_t r11 = 0, r12 = 0, cap = 0, committed = 0;
};

struct Rep {
    StreamPtr st;
    DimensionTree tree;
    Shape dims;
    std::vector<std::vector<DT>> cores;  // non-root cores; cores[0] unused
    std::shared_ptr<RootStore> root;
    int64_t acc = 0;         // slices held locally (this rank's shard)
    int64_t acc_global = 0;  // total tensors streamed (all ranks)
    double eps_rel = 0.0;
    /// sum over the non-root bases of ||U^T U - I||_F (identity bases count 0):
    /// bounds the telescoped loss's error (see telescope_floor_sq)
    double defect = 0.0;

    const DT& core(NodeId id) const {
        return cores.at(static_cast<size_t>(id.layer)).at(static_cast<size_t>(id.pos));
    }
    Index rank(NodeId id) const;
    RankMap ranks() const;
};

struct Context {
    int device = 0;
    StreamPtr st;
    cudaStream_t s = nullptr;
    cudaStream_t s_aux = nullptr;  // side work beside s (full-rank certificates)
    cudaEvent_t aux_ev = nullptr;
    int num_sms = kNumSMs;
    std::string err;
    int64_t launches = 0;
    bool exact_loss = false;
    bool fused = true;
    bool profile = false;
    int tail_kernel = 0;  // HTR_OPT_TAIL_KERNEL
    bool tridiag = true;  // HTR_OPT_EIG_SOLVER: 1 tridiagonal + bisection (default), 0 Jacobi
    double* h_sc = nullptr;  // pinned scalars
    double* h_map = nullptr; // mapped pinned scalars written by kernels (64 doubles)
    double* d_map = nullptr; // its device address
    BufPtr d_sc;             // device scalars
    unsigned int* d_ticket = nullptr;  // last-CTA ticket of the fused tail (kept zero between launches)
    // timing of the fused encode kernel and of the generic GEMMs
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // the stream API's two in-flight slots: done, fused start, fused end
    cudaEvent_t slot_ev[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    double fused_ms = 0.0, gemm_ms = 0.0;
    int64_t fused_calls = 0, gemm_calls = 0;
    // batch-axis sharding over NCCL (dlopen'd), or through a host-staged
    // reducer installed by the caller (htr_context_set_reducer)
    int nranks = 1, rank = 0;
    void* nccl_comm = nullptr;
    htr_host_reduce_fn reducer = nullptr;
    void* reducer_user = nullptr;
    double* h_red = nullptr;  // pinned staging buffer of the host reducer
    int64_t h_red_cap = 0;
    /// Every global quantity goes through allreduce (the context is one rank
    /// of a batch-sharded run).
    bool sharded() const { return nccl_comm != nullptr || reducer != nullptr; }

    /// A Gram computed ahead of its truncation (BHT-l2r reads ||y||^2 off the
    /// first leaf Gram's trace): gram() hands it out once for the same view.
    struct GramHint {
        const double* data = nullptr;
        int mode = -1;
        Shape shape;
        DT G;
    } gram_hint;

    explicit Context(int dev);
    ~Context();

    BufPtr alloc(int64_t n) { return std::make_shared<Buf>(st, n); }
    DT tensor(const Shape& shape) {
        DT t;
        t.shape = shape;
        t.buf = alloc(htrise::shape_product(shape));
        return t;
    }
    /// Sum n doubles over all ranks in place (no-op on one rank).
    void allreduce(double* d, int64_t n);
    /// Copy n device doubles to host (synchronises the stream).
    void fetch(const double* d, int64_t n, double* host);
};

// ---- building blocks -------------------------------------------------------
void run_gemm(Context& c, const GemmDesc& d);
/// out = t x_mode M with M(q, j) = Mp[q*smq + j*smj] (q < Q); written to
/// `dst` (caller memory, out.size() doubles) when given.
DT mode_mul(Context& c, const DT& t, int mode, const double* Mp, int64_t Q, int64_t smq, int64_t smj,
            double* dst = nullptr);
/// Sum over the fibres of (t - U (U^T t)) along `mode`, given coeff = U^T t;
/// result added into the device scalar `slot`.
void residual_energy(Context& c, const DT& t, int mode, const double* U, int64_t r, const DT& coeff,
                     double* slot);
/// Gram of the mode-`mode` unfolding (extent x extent), all-reduced.
DT gram(Context& c, const DT& t, int mode, bool reduce = true);
/// ||x||^2 (all-reduced) and the non-finite flag.
void norm_sq(Context& c, const double* x, int64_t n, double* ysq, bool* nonfinite, bool reduce = true);

struct Truncation {
    DT u;  // rows x rank
    int64_t rank = 0;
    double discarded = 0.0;
    std::vector<double> sigma;  // retained singular values
};
/// Gram (q x q) of W^T M for a device matrix W (rows x q, col-major): lets a
/// truncation re-measure a subspace against the matrix M itself.
using ProjectedGram = std::function<DT(const double* W, int64_t q)>;
/// Error-truncated basis of a symmetric Gram (truncated_svd.hpp:53-100 on the
/// matrix whose Gram this is). k = min(rows, cols). The Gram's eigenvalues
/// carry an absolute rounding error ~u * Lambda, Lambda = max(lambda_max,
/// `noise_scale`); `noise_scale` is the norm of the Gram this one was derived
/// from by subtraction (the unprojected Gram of a residual Gram), 0 for a
/// plain Gram. When the tolerance sits near that floor (eps^2 < 1e-7 Lambda)
/// the eigenvalues below 1e-6 Lambda are re-measured through `refine` (a
/// second Gram of the projection of M onto that subspace), which resolves
/// singular values down to ~u sigma_max like the reference's direct SVD.
Truncation truncate_gram(Context& c, const DT& G, int64_t rows, int64_t cols, double eps_abs, int64_t min_rank,
                         const ProjectedGram& refine = nullptr, double noise_scale = 0.0);
/// Refiner for a plain unfolding of `t` along `mode`.
ProjectedGram unfolding_refiner(Context& c, const DT& t, int mode, bool reduce = true);

/// Basis matrix view (alpha x r) of a non-root core (bht.hpp:81-86).
struct Basis {
    const double* p;
    int64_t alpha, r;
};
/// Unfoldings taller than this (rows > cols, one rank) are truncated through
/// their column-side Gram.
constexpr int64_t kColumnSideRows = 1024;
/// Error-truncated basis of the mode-`mode` unfolding of t, or with `old`
/// of its residual (I - U U^T) t_(mode) (compute_residual, ht_rise.hpp:31-38).
/// cols_global = the unfolding's column count over all ranks; `sharded`
/// false for a rank-local matrix (no all-reduce).
/// any_basis_when_full: the caller needs only the retained subspace (a
/// BHT-l2r node basis), so when the unfolding is certified full rank
/// (lambda_min of its Gram above eps_abs^2 with margin, by a Cholesky test)
/// the identity is returned without an eigensolve. The reference's rank rule
/// keeps every direction then (truncated_svd.hpp:78-93: the tail from
/// r = rows - 1 is sigma_min^2 > eps^2), and any orthonormal basis of the
/// full space spans the same subspace; `sigma` is left empty.
Truncation truncate_mode(Context& c, const DT& t, int mode, const Basis* old, double eps_abs, int64_t min_rank,
                         int64_t cols_global, bool sharded = true, bool any_basis_when_full = false);
/// truncate_mode (no old basis) of several modes of one tensor, in order;
/// the eigensolves of those on the plain Gram route run as one batched launch.
std::vector<Truncation> truncate_modes(Context& c, const DT& t, const std::vector<int>& modes, double eps_abs,
                                       int64_t min_rank, const std::vector<int64_t>& cols_global, bool sharded = true,
                                       bool any_basis_when_full = false, const std::vector<Basis>* olds = nullptr);

// ---- algorithms --------------------------------------------------------------
struct BuildOut {
    std::shared_ptr<Rep> rep;
    htr_build_report report;
};
BuildOut bht_l2r(Context& c, const DT& y, const DimensionTree& tree, double eps_rel, bool adaptive);

/// The skip test's telescoped loss ||y||^2 - ||latent||^2 carries an
/// absolute error of at most beta ||y||^2, beta = 2 D + 16 u, D the bases'
/// orthonormality defect sum (Rep::defect): the nested projections are exact
/// projectors only up to U^T U - I. Its square root is then within
/// kProjErrorTol ||y|| of the explicit-residual value whenever proj^2 >=
/// telescope_floor_sq(h) ||y||^2 = (beta / (2 kProjErrorTol))^2 ||y||^2;
/// below that the loss is re-measured as ||y - decode(latent)||^2.
constexpr double kProjErrorTol = 1e-9;
double telescope_floor_sq(const Rep& h);
/// Rep::defect of every non-root basis (one launch + one read-back).
void measure_defect(Context& c, Rep& h);
/// ||decode(latent) - y||^2 summed over all ranks.
double residual_sq_global(Context& c, const Rep& h, const DT& latent, const DT& y);

struct EncodeOut {
    DT latent;
    double ysq = 0.0;       // ||y||^2 (global)
    double proj_sq = 0.0;   // projection error^2
    bool fused = false;
    bool exact = false;
    bool nonfinite = false;
    int64_t gbatch = 0;     // samples of this batch over all ranks (same all-reduce)
    bool scan_valid = false;  // deferred: sc[1] carries the non-finite flag of a full ||y||^2 scan
};
/// `latent_target`, when given, is where the fused tail writes the latent if
/// it runs (a view of the root store's next free slices): a skip decision
/// then only commits it.
/// With `sc_deferred` (16 device doubles) the encode only enqueues its work:
/// ||y||^2 -> sc[0], the non-finite flag -> sc[1] (when scan_valid),
/// ||latent||^2 -> sc[2]; the caller all-reduces and reads them back (the
/// stream API's pipelining). EncodeOut then carries the latent only.
EncodeOut encode(Context& c, const Rep& h, const DT& y, bool exact, const DT* latent_target = nullptr,
                 double* sc_deferred = nullptr);

struct UpdateOut {
    std::shared_ptr<Rep> rep;
    htr_update_report report;
};
UpdateOut ht_rise_update(Context& c, const Rep& h, const DT& y, double eps_override, bool adaptive);

/// The skip-path encode of a 3-way (1,(2,3)) batch as two launches (fused3 +
/// tail3), ||y||^2 -> sc[0] and ||latent||^2 -> sc[2]. false (nothing
/// launched) outside the fused kernels' shapes and ranks.
/// host_out (device address of mapped host memory, or null) receives the
/// same two scalars.
bool launch_skip_encode3(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc, DT* latent,
                         cudaEvent_t ev0, cudaEvent_t ev1, double* host_out = nullptr);
/// The same for 8-way balanced trees with extents 8 and ranks 4 (two
/// 4-leaf subtree launches, config 4).
bool launch_skip_encode8(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc, DT* latent,
                         cudaEvent_t ev0, cudaEvent_t ev1, double* host_out = nullptr);
/// The same for balanced 4-way trees ((1,2),(3,4)) whose leading slabs fit the
/// fused leaf kernel (config 3): fused3 over modes 0, 1 + the per-sample tail.
bool launch_skip_encode4(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc, DT* latent,
                         cudaEvent_t ev0, cudaEvent_t ev1, double* host_out = nullptr);
/// Whichever fused skip-path encode applies (3-, 4- or 8-way); false when none.
bool launch_skip_encode_fused(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc,
                              DT* latent, cudaEvent_t ev0, cudaEvent_t ev1, double* host_out = nullptr);

/// A stream of updates h -> h1 -> ... -> hn, identical to n ht_rise_update
/// calls (extension: the reference's caller loops over batches, main.cpp).
/// While batch i's skip decision is read back, batch i+1's skip-path encode
/// is already queued against the same bases (a skip leaves them unchanged);
/// when batch i expands, that speculative work is discarded and batch i+1
/// re-runs against the new bases. batch_of(i) supplies batch i (called once
/// per batch, in order).
std::vector<UpdateOut> ht_rise_update_many(Context& c, const std::shared_ptr<Rep>& h, int64_t n,
                                           const std::function<DT(int64_t)>& batch_of, double eps_override,
                                           bool adaptive);

/// bht.hpp:406-456; the result lands in `dst` (caller device memory) when given.
DT decode(Context& c, const Rep& h, const DT& latent, double* dst = nullptr);
/// sum (decode(latent) - y)^2 over this rank's samples into the device scalar
/// `out`, without materialising the reconstruction where the fused decode
/// kernel applies (relative_test_error, metrics.hpp:218-237).
/// out[0] = ||y - decode(latent)||^2 (enqueued). With host_out (device address
/// of mapped host memory) the fused reconstruction kernel also writes the
/// value there; returns whether it did (false: the generic chain ran and the
/// caller copies out[0] back).
bool decode_residual_sq(Context& c, const Rep& h, const DT& latent, const DT& y, double* out,
                        double* host_out = nullptr);

/// Append latent slices [r11, r12, N] to a representation's root (value
/// semantics: returns the new root view).
void append_root(Context& c, Rep& out, const Rep& in, const DT& latent);

// validation shared with the C-ABI
DimensionTree tree_from_nodes(const htr_node* nodes, int64_t n);
void nodes_from_tree(const DimensionTree& t, std::vector<htr_node>& out);
void check_batch_input(const Shape& y_shape, const DimensionTree& tree, const Shape* dims, const char* who);

}  // namespace htr
