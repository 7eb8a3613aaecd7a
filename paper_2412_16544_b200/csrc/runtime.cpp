// htrise-b200 native runtime: the reference's Alg. 1 (BHT-l2r, bht.hpp:251-350)
// and Alg. 2 (HT-RISE, ht_rise.hpp:99-186) orchestrated on device-resident
// data. The host walks the dimension tree (integer metadata) and enqueues
// kernels on one stream; the only host round trips are the scalars that
// decide control flow (ranks after a truncation, the skip test).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <tuple>

#include "runtime.hpp"

namespace htr {

void raise(htr_status code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what, int line) {
    // HTR_DEBUG_SYNC=1: synchronise after every checked call so a faulting
    // kernel is reported at the launch site that queued it
    static const bool debug_sync = [] {
        const char* v = std::getenv("HTR_DEBUG_SYNC");
        return v && v[0] == '1';
    }();
    if (e == cudaSuccess && debug_sync) e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
        raise(HTR_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what + " (line " +
                                std::to_string(line) + ")");
}

Stream::Stream(int dev) : device(dev) {
    HTR_CUDA(cudaSetDevice(dev));
    HTR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
}
Stream::~Stream() {
    if (s) {
        cudaStreamSynchronize(s);
        for (auto& bin : bins)
            for (double* p : bin) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
}

int Stream::size_class(int64_t n) {
    if (n <= 0 || n > (int64_t{1} << kMaxClass)) return -1;
    int c = kMinClass;
    while ((int64_t{1} << c) < n) ++c;
    return c;
}

double* Stream::take(int cls) {
    std::lock_guard<std::mutex> g(mu);
    auto& bin = bins[cls];
    if (bin.empty()) return nullptr;
    double* p = bin.back();
    bin.pop_back();
    cached_bytes -= sizeof(double) << cls;
    return p;
}

bool Stream::give(int cls, double* p) {
    std::lock_guard<std::mutex> g(mu);
    const size_t bytes = sizeof(double) << cls;
    if (cached_bytes + bytes > kCacheCapBytes) return false;
    bins[cls].push_back(p);
    cached_bytes += bytes;
    return true;
}

Buf::Buf(StreamPtr st_, int64_t n_) : st(std::move(st_)), n(n_) {
    if (n <= 0) return;
    cls = Stream::size_class(n);
    if (cls >= 0 && (p = st->take(cls)) != nullptr) return;
    const size_t doubles = cls >= 0 ? size_t{1} << cls : static_cast<size_t>(n);
    HTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), doubles * sizeof(double), st->s));
}
Buf::~Buf() {
    if (!p || !owned) return;
    if (cls >= 0 && st->give(cls, p)) return;
    cudaFreeAsync(p, st->s);
}

Index Rep::rank(NodeId id) const {
    const TreeNode& n = tree.node(id);
    if (n.kind == NodeKind::Root) raise(HTR_ERR_INVALID_ARGUMENT, "rank: root has no own rank");
    const DT& c = core(id);
    return n.kind == NodeKind::Leaf ? c.shape[1] : c.shape[2];
}

RankMap Rep::ranks() const {
    RankMap r;
    for (Index l = 1; l <= tree.depth(); ++l)
        for (const TreeNode& n : tree.layer(l)) r[n.id] = rank(n.id);
    return r;
}

// ---------------------------------------------------------------------------
// NCCL (dlopen'd so that the process uses whichever libnccl torch loaded)
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (!api.lib) {
        api.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.lib) raise(HTR_ERR_RUNTIME, std::string("cannot load libnccl.so.2: ") + dlerror());
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.lib, "ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.lib, "ncclCommInitRank"));
        api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(api.lib, "ncclAllReduce"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.lib, "ncclCommDestroy"));
        api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(api.lib, "ncclGetErrorString"));
        if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy)
            raise(HTR_ERR_RUNTIME, "libnccl.so.2 lacks required symbols");
    }
    return api;
}
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* m = nccl().getErrorString ? nccl().getErrorString(r) : "?";
        raise(HTR_ERR_RUNTIME, std::string("NCCL error ") + m + " at " + what);
    }
}
}  // namespace

void comm_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, 128);
}

void set_reducer(Context& c, htr_host_reduce_fn fn, void* user, int nranks, int rank) {
    if (!fn) raise(HTR_ERR_INVALID_ARGUMENT, "set_reducer: null reduce function");
    if (nranks < 1 || rank < 0 || rank >= nranks) raise(HTR_ERR_INVALID_ARGUMENT, "bad nranks/rank for set_reducer");
    if (c.sharded()) raise(HTR_ERR_INVALID_ARGUMENT, "context already has a communicator");
    c.reducer = fn;
    c.reducer_user = user;
    c.nranks = nranks;
    c.rank = rank;
}

void comm_init(Context& c, const uint8_t uid[128], int nranks, int rank) {
    // An explicit call always builds a communicator, a single-rank one
    // included: every reduction then goes through NCCL exactly as at N > 1.
    if (nranks < 1 || rank < 0 || rank >= nranks) raise(HTR_ERR_INVALID_ARGUMENT, "bad nranks/rank for init_comm");
    if (c.sharded()) raise(HTR_ERR_INVALID_ARGUMENT, "context already has a communicator");
    ncclUniqueId id;
    std::memcpy(&id, uid, 128);
    ncclComm_t comm;
    HTR_CUDA(cudaSetDevice(c.device));
    nccl_check(nccl().commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    c.nccl_comm = comm;
    c.nranks = nranks;
    c.rank = rank;
}

Context::Context(int dev) : device(dev) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        raise(HTR_ERR_NO_DEVICE, "htrise-b200 needs a CUDA device (sm_100a); none is visible");
    if (dev < 0 || dev >= count) raise(HTR_ERR_NO_DEVICE, "device index out of range");
    st = std::make_shared<Stream>(dev);
    s = st->s;
    HTR_CUDA(cudaStreamCreateWithFlags(&s_aux, cudaStreamNonBlocking));
    HTR_CUDA(cudaEventCreateWithFlags(&aux_ev, cudaEventDisableTiming));
    HTR_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    cudaMemPool_t pool;
    HTR_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    HTR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    HTR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_sc), 1024 * sizeof(double)));
    HTR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_map), 64 * sizeof(double), cudaHostAllocMapped));
    HTR_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_map), h_map, 0));
    d_sc = alloc(1024);
    HTR_CUDA(cudaMalloc(reinterpret_cast<void**>(&d_ticket), sizeof(unsigned int)));
    HTR_CUDA(cudaMemset(d_ticket, 0, sizeof(unsigned int)));
    for (auto& e : ev) HTR_CUDA(cudaEventCreate(&e));
    for (auto& se : slot_ev) {
        HTR_CUDA(cudaEventCreateWithFlags(&se[0], cudaEventDisableTiming));
        HTR_CUDA(cudaEventCreate(&se[1]));
        HTR_CUDA(cudaEventCreate(&se[2]));
    }
}

Context::~Context() {
    if (s) cudaStreamSynchronize(s);
    if (s_aux) {
        cudaStreamSynchronize(s_aux);
        cudaStreamDestroy(s_aux);
    }
    if (aux_ev) cudaEventDestroy(aux_ev);
    if (nccl_comm) nccl().commDestroy(static_cast<ncclComm_t>(nccl_comm));
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    for (auto& se : slot_ev)
        for (auto& e : se)
            if (e) cudaEventDestroy(e);
    if (h_red) cudaFreeHost(h_red);
    if (h_sc) cudaFreeHost(h_sc);
    if (h_map) cudaFreeHost(h_map);
    if (d_ticket) cudaFree(d_ticket);
}

void Context::allreduce(double* d, int64_t n) {
    if (n == 0) return;
    if (reducer) {
        // host-staged: the partial sums reach the caller's transport through
        // pinned memory; the stream is drained first, so no kernel of this
        // rank waits on another rank's device work
        if (n > h_red_cap) {
            if (h_red) HTR_CUDA(cudaFreeHost(h_red));
            h_red = nullptr;
            HTR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_red), static_cast<size_t>(n) * sizeof(double)));
            h_red_cap = n;
        }
        HTR_CUDA(cudaMemcpyAsync(h_red, d, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
        HTR_CUDA(cudaStreamSynchronize(s));
        if (reducer(h_red, n, reducer_user) != 0) raise(HTR_ERR_RUNTIME, "host reducer failed");
        HTR_CUDA(cudaMemcpyAsync(d, h_red, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s));
        // (the next allreduce drains the stream before reusing h_red)
        return;
    }
    if (!nccl_comm) return;
    nccl_check(nccl().allReduce(d, d, static_cast<size_t>(n), ncclDouble, ncclSum,
                                static_cast<ncclComm_t>(nccl_comm), s),
               "ncclAllReduce");
}

void Context::fetch(const double* d, int64_t n, double* host) {
    if (n <= 0) return;
    HTR_CUDA(cudaMemcpyAsync(host, d, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
    HTR_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// building blocks
// ---------------------------------------------------------------------------

void run_gemm(Context& c, const GemmDesc& d) {
    if (d.N1 * d.N2 >= (int64_t{1} << 31) || d.K1 * d.K2 >= (int64_t{1} << 31))
        raise(HTR_ERR_RUNTIME, "contraction extent exceeds 2^31 elements; split the batch");
    const int64_t ws = gemm_workspace_doubles(d, c.num_sms);
    BufPtr w = ws > 0 ? c.alloc(ws) : nullptr;
    launch_gemm(d, w ? w->p : nullptr, c.num_sms, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
}

namespace {
struct Split {
    int64_t I = 1, J = 1, O = 1;
};
Split split_at(const Shape& s, int mode) {
    Split p;
    for (int k = 0; k < mode; ++k) p.I *= s[static_cast<size_t>(k)];
    p.J = s[static_cast<size_t>(mode)];
    for (size_t k = static_cast<size_t>(mode) + 1; k < s.size(); ++k) p.O *= s[k];
    return p;
}
}  // namespace

DT mode_mul(Context& c, const DT& t, int mode, const double* Mp, int64_t Q, int64_t smq, int64_t smj, double* dst) {
    const Split sp = split_at(t.shape, mode);
    Shape os = t.shape;
    os[static_cast<size_t>(mode)] = Q;
    DT out;
    if (dst) {
        out.shape = os;
        out.buf = std::make_shared<Buf>(c.st, dst, htrise::shape_product(os));
    } else {
        out = c.tensor(os);
    }
    const bool small = sp.J <= 16 && Q <= 16 && sp.I * sp.O >= 4096;
    if (!small && Q >= 32 && Q <= 128 && sp.J <= 32 && sp.I >= 64) {
        // an r -> n expansion (decode): persistent kernel, factor resident
        if (launch_expand(t.data(), sp.I, sp.J, sp.O, Mp, Q, smq, smj, out.data(), c.num_sms, c.s, &c.launches) > 0) {
            HTR_CUDA(cudaGetLastError());
            return out;
        }
    }
    if (!small && Q >= 32 && sp.I > 1 && sp.O > 1 && sp.O <= 65535) {
        // an interior mode producing >= 32 rows (decode's leaf expansions):
        // one plain GEMM per outer index (the (i, o) column map is not a
        // single stride), eligible for the fast kernel
        GemmDesc b;
        b.M = Q; b.N1 = sp.I; b.K1 = sp.J; b.batch = sp.O;
        b.A = Mp; b.sam = smq; b.sak1 = smj;
        b.B = t.data(); b.sbk1 = sp.I; b.sbn1 = 1; b.sbb = sp.I * sp.J;
        b.C = out.data(); b.scm = sp.I; b.scn1 = 1; b.scb = sp.I * Q;
        if (gemm_is_fast(b, c.num_sms)) {
            run_gemm(c, b);
            return out;
        }
    }
    if (small) {
        // tiny extents: streaming kernel (the MMA tiles would be mostly padding)
        if (launch_mode_small(t.data(), sp.I, sp.J, sp.O, Mp, Q, smq, smj, out.data(), nullptr, nullptr, c.num_sms,
                              c.s, &c.launches) > 0) {
            HTR_CUDA(cudaGetLastError());
            return out;
        }
    }
    GemmDesc d;
    d.M = Q;
    d.N1 = sp.I;
    d.N2 = sp.O;
    d.K1 = sp.J;
    d.K2 = 1;
    d.A = Mp;
    d.sam = smq;
    d.sak1 = smj;
    d.B = t.data();
    d.sbk1 = sp.I;
    d.sbn1 = 1;
    d.sbn2 = sp.I * sp.J;
    d.C = out.data();
    d.scm = sp.I;
    d.scn1 = 1;
    d.scn2 = sp.I * Q;
    run_gemm(c, d);
    return out;
}

void residual_energy(Context& c, const DT& t, int mode, const double* U, int64_t r, const DT& coeff,
                     double* slot) {
    // D = t, acc = U * coeff along `mode`: sum (t - U coeff)^2 (bht.hpp:361)
    const Split sp = split_at(t.shape, mode);
    GemmDesc d;
    d.M = sp.J;
    d.N1 = sp.I;
    d.N2 = sp.O;
    d.K1 = r;
    d.A = U;
    d.sam = 1;
    d.sak1 = sp.J;
    d.B = coeff.data();
    d.sbk1 = sp.I;
    d.sbn1 = 1;
    d.sbn2 = sp.I * r;
    d.D = t.data();
    d.scm = sp.I;
    d.scn1 = 1;
    d.scn2 = sp.I * sp.J;
    BufPtr parts = c.alloc(1);
    d.energy_partials = parts->p;  // sized below once the tile plan is known
    const int64_t tiles = gemm_energy_partials(d, c.num_sms);
    parts = c.alloc(tiles);
    d.energy_partials = parts->p;
    launch_gemm(d, nullptr, c.num_sms, c.s, &c.launches);
    launch_sum_partials(parts->p, tiles, slot, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
}

DT gram(Context& c, const DT& t, int mode, bool reduce) {
    if (c.gram_hint.G.buf && c.gram_hint.data == t.data() && c.gram_hint.mode == mode && c.gram_hint.shape == t.shape) {
        DT G = c.gram_hint.G;  // already all-reduced
        c.gram_hint = Context::GramHint{};
        return G;
    }
    c.gram_hint = Context::GramHint{};
    const Split sp = split_at(t.shape, mode);
    DT G = c.tensor({sp.J, sp.J});
    if (c.fused && sp.J <= 8 && sp.I * sp.J * sp.O >= (int64_t{1} << 20) && gram_small_supported(sp.I, sp.J, sp.O)) {
        // few rows (c4's 8-extent modes): one column per thread, registers
        BufPtr parts = c.alloc(gram_small_partials(c.num_sms));
        launch_gram_small(t.data(), sp.I, sp.J, sp.O, parts->p, G.data(), c.num_sms, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        if (reduce) c.allreduce(G.data(), sp.J * sp.J);
        return G;
    }
    if (c.fused && sp.I == 1 && sp.J > 32 && sp.J * sp.O >= (int64_t{1} << 16) &&
        gram_mode0_supported(t.data(), sp.J, sp.O)) {
        // mode 0 (rows contiguous), 33..128 rows: shared-memory column chunks on DMMA
        BufPtr parts = c.alloc(gram_stream_partials(sp.J, c.num_sms));
        launch_gram_mode0(t.data(), sp.J, sp.O, parts->p, G.data(), c.num_sms, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        if (reduce) c.allreduce(G.data(), sp.J * sp.J);
        return G;
    }
    if (c.fused && sp.J >= 9 && sp.J <= 32 && gram_mid_supported(sp.I, sp.J, sp.O) &&
        !(sp.J >= 24 && sp.I * sp.J * sp.O >= (int64_t{1} << 22) && gram_stream_supported(t.data(), sp.I, sp.J, sp.O))) {
        // 9..32 rows, any mode: DMMA over 4-column k-steps (the streaming
        // kernel keeps the large >= 24-row modes it supports)
        BufPtr parts = c.alloc(gram_mid_partials(c.num_sms));
        launch_gram_mid(t.data(), sp.I, sp.J, sp.O, parts->p, G.data(), c.num_sms, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        if (reduce) c.allreduce(G.data(), sp.J * sp.J);
        return G;
    }
    if (c.fused && sp.J >= 24 && sp.I * sp.J * sp.O >= (int64_t{1} << 22) &&
        gram_stream_supported(t.data(), sp.I, sp.J, sp.O)) {
        // large unfolding of a mode >= 1 with >= 24 rows: the streaming
        // lower-triangle kernel (its 32 x 32 warp blocks would be mostly
        // padding for fewer rows)
        BufPtr parts = c.alloc(gram_stream_partials(sp.J, c.num_sms));
        if (launch_gram_stream(t.data(), sp.I, sp.J, sp.O, parts->p, G.data(), c.num_sms, c.s, &c.launches) > 0) {
            HTR_CUDA(cudaGetLastError());
            if (reduce) c.allreduce(G.data(), sp.J * sp.J);
            return G;
        }
    }
    GemmDesc d;
    d.M = sp.J;
    d.N1 = sp.J;
    d.N2 = 1;
    d.K1 = sp.I;
    d.K2 = sp.O;
    d.A = t.data();
    d.sam = sp.I;
    d.sak1 = 1;
    d.sak2 = sp.I * sp.J;
    d.B = t.data();
    d.sbk1 = 1;
    d.sbk2 = sp.I * sp.J;
    d.sbn1 = sp.I;
    d.C = G.data();
    d.scm = 1;
    d.scn1 = sp.J;
    d.symmetric = true;
    run_gemm(c, d);
    if (reduce) c.allreduce(G.data(), sp.J * sp.J);
    return G;
}

void norm_sq(Context& c, const double* x, int64_t n, double* ysq, bool* nonfinite, bool reduce) {
    BufPtr parts = c.alloc(kReduceBlocks);
    launch_sumsq(x, n, parts->p, c.d_sc->p, c.s, &c.launches);
    if (reduce) c.allreduce(c.d_sc->p, 2);
    c.fetch(c.d_sc->p, 2, c.h_sc);
    *ysq = c.h_sc[0];
    if (nonfinite) *nonfinite = c.h_sc[1] != 0.0;
}

ProjectedGram unfolding_refiner(Context& c, const DT& t, int mode);

Truncation truncate_eig(Context& c, const BufPtr& lam, const BufPtr& V, int64_t rows, int64_t cols, double eps_abs,
                        int64_t min_rank, const ProjectedGram& refine, double noise_scale);

/// Relative tolerance below which a truncation's small eigenvalues are
/// re-measured (eps^2 < refine_threshold(n) * lambda_max): the Gram's
/// eigenvalues carry an absolute error ~n u lambda_max each, so a tail sum of
/// up to n of them is uncertain by ~n^2 u lambda_max; above 1e5 times that
/// the rank rule's decision cannot move, below it the tail is re-measured
/// through a projected Gram (then resolved to ~u sigma_max like the
/// reference's direct SVD). Capped at 1e-7 (the former fixed threshold).
double refine_threshold(int64_t n) {
    const double nn = static_cast<double>(std::max<int64_t>(n, 1));
    return std::min(1e-7, 1e5 * nn * nn * 0x1p-53);
}

/// Every eigenpair of a symmetric n x n G (lambda descending, V n x n): the
/// tridiagonal route with all n vectors for small n (the machine-floor
/// refinement of small Grams), else the Jacobi solver. `work` holds 2 n^2
/// doubles (Jacobi).
void eig_full(Context& c, const double* G, int64_t n, double* lam, double* V, double* work) {
    if (c.tridiag && n <= kTriFullMaxN) {
        BufPtr W = c.alloc(tridiag_workspace_doubles(n));
        BufPtr info = c.alloc(4);
        launch_fill(info->p, 4, 1.0, c.s, &c.launches);  // info[2] != 0: not the zero-input case
        double* wp = W->p;
        launch_tridiag_eigvals(&G, &n, &lam, &wp, 1, c.s, &c.launches);
        const double* wc = W->p;
        const double* ip = info->p;
        launch_tridiag_vectors(&wc, &ip, &n, &n, &V, 1, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        return;
    }
    launch_jacobi_eig(G, n, lam, V, work, c.s, &c.launches);
}

/// A Gram reduced to tridiagonal form with all its eigenvalues (descending)
/// on the device (k_tridiag.cu); W keeps the reflectors for the vectors.
struct TriSolve {
    BufPtr lam, W;
    int64_t n = 0;
};

TriSolve tri_alloc(Context& c, int64_t n) {
    TriSolve t;
    t.n = n;
    t.lam = c.alloc(n);
    t.W = c.alloc(tridiag_workspace_doubles(n));
    return t;
}

Truncation truncate_jacobi(Context& c, const DT& G, int64_t rows, int64_t cols, double eps_abs, int64_t min_rank,
                           const ProjectedGram& refine, double noise_scale);

/// The rank rule (truncated_svd.hpp:74-99) on a tridiagonal solve's
/// eigenvalues and the retained eigenvectors. A truncation whose tolerance
/// sits at the Gram's rounding floor re-measures its small eigenvalues
/// through `refine`, which needs every eigenvector: that (rare) case takes
/// the Jacobi solver on the untouched Gram instead.
Truncation finish_tri(Context& c, const TriSolve& ts, const DT& G, int64_t rows, int64_t cols, double eps_abs,
                      int64_t min_rank, const ProjectedGram& refine, double noise_scale) {
    const int64_t n = rows;
    const int64_t k = std::min(rows, cols);
    if (refine) {
        std::vector<double> lh(static_cast<size_t>(n));
        c.fetch(ts.lam->p, n, lh.data());
        const double lmax = std::max({lh[0], noise_scale, 0.0});
        if (lmax > 0.0 && eps_abs * eps_abs < refine_threshold(n) * lmax) {
            int64_t s0 = 0;
            while (s0 < n && lh[static_cast<size_t>(s0)] >= 1e-6 * lmax) ++s0;
            if (s0 < n) return truncate_jacobi(c, G, rows, cols, eps_abs, min_rank, refine, noise_scale);
        }
    }
    BufPtr info = c.alloc(4);
    launch_rank_rule(ts.lam->p, k, n, eps_abs, min_rank, nullptr, info->p, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    double h[4];
    c.fetch(info->p, 3, h);
    Truncation t;
    t.rank = static_cast<int64_t>(h[0]);
    t.discarded = h[1];
    const bool zero = h[2] == 0.0;
    if (t.rank > 0) {
        std::vector<double> l(static_cast<size_t>(t.rank));
        c.fetch(ts.lam->p, t.rank, l.data());
        t.sigma.resize(static_cast<size_t>(t.rank));
        for (int64_t i = 0; i < t.rank; ++i)
            t.sigma[static_cast<size_t>(i)] = zero ? 0.0 : std::sqrt(std::max(0.0, l[static_cast<size_t>(i)]));
    }
    t.u = c.tensor({rows, t.rank});
    if (t.rank > 0) {
        const double* Wp = ts.W->p;
        const double* ip = info->p;
        double* up = t.u.data();
        launch_tridiag_vectors(&Wp, &ip, &n, &t.rank, &up, 1, c.s, &c.launches);
        if (!zero) {  // CholeskyQR2 polish (as truncate_eig)
            BufPtr oinfo = c.alloc(4);
            BufPtr work = c.alloc(t.rank * t.rank + 16);
            launch_orthonormalize_new(nullptr, rows, 0, t.u.data(), t.rank, oinfo->p, work->p, c.s, &c.launches);
        }
    }
    HTR_CUDA(cudaGetLastError());
    return t;
}

/// finish_tri for the nodes of one layer at once: every node's rank rule is
/// enqueued before the first result is read back, and the retained
/// eigenvectors of all nodes are formed by ONE launch (a CTA per node) instead
/// of one launch per node behind a host round trip each (c1's four leaves:
/// 4 x 76 us of single-CTA launches -> one). Results equal finish_tri's bit
/// for bit.
std::vector<Truncation> finish_tri_batch(Context& c, const std::vector<TriSolve>& ts, const std::vector<DT>& G,
                                         const std::vector<int64_t>& rows, const std::vector<int64_t>& cols,
                                         double eps_abs, int64_t min_rank, const std::vector<ProjectedGram>& refine,
                                         const std::vector<double>& noise) {
    const size_t m = ts.size();
    std::vector<Truncation> out(m);
    if (m > 200) {  // (the pinned staging block holds 4 doubles per node) one by one
        for (size_t j = 0; j < m; ++j)
            out[j] = finish_tri(c, ts[j], G[j], rows[j], cols[j], eps_abs, min_rank, refine[j], noise[j]);
        return out;
    }
    std::vector<char> done(m, 0);
    // every node's eigenvalues in one read-back (pinned staging, one stream
    // synchronisation for the layer instead of one per node)
    std::vector<std::vector<double>> lam(m);
    {
        int64_t total = 0;
        for (size_t j = 0; j < m; ++j) total += rows[j];
        const bool staged = total <= 896;  // h_sc holds 1024 doubles; [960..) belongs to the stream slots
        int64_t off = 0;
        for (size_t j = 0; j < m; ++j) {
            lam[j].resize(static_cast<size_t>(rows[j]));
            if (staged) {
                HTR_CUDA(cudaMemcpyAsync(c.h_sc + off, ts[j].lam->p, sizeof(double) * static_cast<size_t>(rows[j]),
                                         cudaMemcpyDeviceToHost, c.s));
                off += rows[j];
            } else {
                c.fetch(ts[j].lam->p, rows[j], lam[j].data());
            }
        }
        if (staged) {
            HTR_CUDA(cudaStreamSynchronize(c.s));
            off = 0;
            for (size_t j = 0; j < m; ++j) {
                std::copy(c.h_sc + off, c.h_sc + off + rows[j], lam[j].begin());
                off += rows[j];
            }
        }
    }
    for (size_t j = 0; j < m; ++j) {
        if (!refine[j]) continue;
        const int64_t n = rows[j];
        const std::vector<double>& lh = lam[j];
        const double lmax = std::max({lh[0], noise[j], 0.0});
        if (lmax > 0.0 && eps_abs * eps_abs < refine_threshold(n) * lmax) {
            int64_t s0 = 0;
            while (s0 < n && lh[static_cast<size_t>(s0)] >= 1e-6 * lmax) ++s0;
            if (s0 < n) {
                out[j] = truncate_jacobi(c, G[j], rows[j], cols[j], eps_abs, min_rank, refine[j], noise[j]);
                done[j] = 1;
            }
        }
    }
    std::vector<BufPtr> infos(m);
    size_t pending = 0;
    for (size_t j = 0; j < m; ++j) {
        if (done[j]) continue;
        infos[j] = c.alloc(4);
        launch_rank_rule(ts[j].lam->p, std::min(rows[j], cols[j]), rows[j], eps_abs, min_rank, nullptr, infos[j]->p, c.s,
                         &c.launches);
        HTR_CUDA(cudaMemcpyAsync(c.h_sc + 4 * pending, infos[j]->p, 3 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
        ++pending;
    }
    HTR_CUDA(cudaGetLastError());
    HTR_CUDA(cudaStreamSynchronize(c.s));
    std::vector<char> zero(m, 0);
    std::vector<const double*> Wp, ip;
    std::vector<int64_t> nn, rr;
    std::vector<double*> up;
    size_t slot = 0;
    for (size_t j = 0; j < m; ++j) {
        if (done[j]) continue;
        const double* h = c.h_sc + 4 * slot++;
        Truncation& t = out[j];
        t.rank = static_cast<int64_t>(h[0]);
        t.discarded = h[1];
        zero[j] = h[2] == 0.0;
        if (t.rank > 0) {
            // (the rank rule does not change the eigenvalues read above)
            t.sigma.resize(static_cast<size_t>(t.rank));
            for (int64_t i = 0; i < t.rank; ++i)
                t.sigma[static_cast<size_t>(i)] = zero[j] ? 0.0 : std::sqrt(std::max(0.0, lam[j][static_cast<size_t>(i)]));
        }
        t.u = c.tensor({rows[j], t.rank});
        if (t.rank > 0) {
            Wp.push_back(ts[j].W->p);
            ip.push_back(infos[j]->p);
            nn.push_back(rows[j]);
            rr.push_back(t.rank);
            up.push_back(t.u.data());
        }
    }
    if (!Wp.empty())
        launch_tridiag_vectors(Wp.data(), ip.data(), nn.data(), rr.data(), up.data(), static_cast<int>(Wp.size()), c.s,
                               &c.launches);
    for (size_t j = 0; j < m; ++j) {
        if (done[j] || out[j].rank <= 0 || zero[j]) continue;
        BufPtr oinfo = c.alloc(4);  // CholeskyQR2 polish (as finish_tri)
        BufPtr work = c.alloc(out[j].rank * out[j].rank + 16);
        launch_orthonormalize_new(nullptr, rows[j], 0, out[j].u.data(), out[j].rank, oinfo->p, work->p, c.s, &c.launches);
    }
    HTR_CUDA(cudaGetLastError());
    return out;
}

Truncation truncate_gram(Context& c, const DT& G, int64_t rows, int64_t cols, double eps_abs, int64_t min_rank,
                         const ProjectedGram& refine, double noise_scale) {
    if (c.tridiag && tridiag_supported(rows)) {
        TriSolve ts = tri_alloc(c, rows);
        const double* gp = G.data();
        double* lp = ts.lam->p;
        double* wp = ts.W->p;
        launch_tridiag_eigvals(&gp, &rows, &lp, &wp, 1, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        return finish_tri(c, ts, G, rows, cols, eps_abs, min_rank, refine, noise_scale);
    }
    return truncate_jacobi(c, G, rows, cols, eps_abs, min_rank, refine, noise_scale);
}

Truncation truncate_jacobi(Context& c, const DT& G, int64_t rows, int64_t cols, double eps_abs, int64_t min_rank,
                           const ProjectedGram& refine, double noise_scale) {
    const int64_t n = rows;
    if (n > kJacobiMaxN)
        raise(HTR_ERR_RUNTIME, "truncation of a " + std::to_string(n) + "-row unfolding " +
                                   (c.tridiag && tridiag_supported(n)
                                        ? "at a tolerance near the Gram's rounding floor (re-measuring its small "
                                          "eigenvalues needs every eigenvector) exceeds the " +
                                              std::to_string(kJacobiMaxN) + "-row limit of that path"
                                        : "exceeds the device eigensolver's " + std::to_string(kJacobiMaxN) +
                                              "-row limit"));
    BufPtr lam = c.alloc(n);
    BufPtr V = c.alloc(n * n);
    BufPtr work = c.alloc(2 * n * n);
    eig_full(c, G.data(), n, lam->p, V->p, work->p);
    HTR_CUDA(cudaGetLastError());
    return truncate_eig(c, lam, V, rows, cols, eps_abs, min_rank, refine, noise_scale);
}

Truncation truncate_eig(Context& c, const BufPtr& lam, const BufPtr& V, int64_t rows, int64_t cols, double eps_abs,
                        int64_t min_rank, const ProjectedGram& refine, double noise_scale) {
    const int64_t n = rows;
    const int64_t k = std::min(rows, cols);
    BufPtr info = c.alloc(4);
    if (refine) {
        std::vector<double> lh(static_cast<size_t>(n));
        c.fetch(lam->p, n, lh.data());
        const double lmax = std::max({lh[0], noise_scale, 0.0});
        if (lmax > 0.0 && eps_abs * eps_abs < refine_threshold(n) * lmax) {
            int64_t s0 = 0;
            while (s0 < n && lh[static_cast<size_t>(s0)] >= 1e-6 * lmax) ++s0;
            const int64_t q = n - s0;
            if (q > 0) {
                double* W = V->p + n * s0;  // eigenvectors of the small eigenvalues
                DT G2 = refine(W, q);
                BufPtr mu = c.alloc(q);
                BufPtr Z = c.alloc(q * q);
                BufPtr work2 = c.alloc(2 * q * q);
                eig_full(c, G2.data(), q, mu->p, Z->p, work2->p);
                HTR_CUDA(cudaMemcpyAsync(lam->p + s0, mu->p, sizeof(double) * static_cast<size_t>(q),
                                         cudaMemcpyDeviceToDevice, c.s));
                BufPtr WZ = c.alloc(n * q);
                GemmDesc d;  // WZ = W Z
                d.M = n; d.N1 = q; d.K1 = q;
                d.A = W; d.sam = 1; d.sak1 = n;
                d.B = Z->p; d.sbk1 = 1; d.sbn1 = q;
                d.C = WZ->p; d.scm = 1; d.scn1 = n;
                run_gemm(c, d);
                HTR_CUDA(cudaMemcpyAsync(W, WZ->p, sizeof(double) * static_cast<size_t>(n * q), cudaMemcpyDeviceToDevice,
                                         c.s));
                HTR_CUDA(cudaGetLastError());
            }
        }
    }
    launch_rank_rule(lam->p, k, n, eps_abs, min_rank, nullptr, info->p, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    double h[4];
    c.fetch(info->p, 3, h);
    Truncation t;
    t.rank = static_cast<int64_t>(h[0]);
    t.discarded = h[1];
    const bool zero = h[2] == 0.0;
    if (t.rank > 0) {
        std::vector<double> l(static_cast<size_t>(t.rank));
        c.fetch(lam->p, t.rank, l.data());
        t.sigma.resize(static_cast<size_t>(t.rank));
        for (int64_t i = 0; i < t.rank; ++i)
            t.sigma[static_cast<size_t>(i)] = zero ? 0.0 : std::sqrt(std::max(0.0, l[static_cast<size_t>(i)]));
    }
    t.u = c.tensor({rows, t.rank});
    launch_take_columns(V->p, n, t.rank, t.u.data(), info->p, c.s, &c.launches);
    if (t.rank > 0 && !zero) {
        // CholeskyQR2 of the retained eigenvectors: the span is unchanged and
        // U^T U - I drops to the u level (it bounds the telescoped skip
        // test's error, telescope_floor_sq)
        BufPtr oinfo = c.alloc(4);
        BufPtr work = c.alloc(t.rank * t.rank + 16);
        launch_orthonormalize_new(nullptr, rows, 0, t.u.data(), t.rank, oinfo->p, work->p, c.s, &c.launches);
    }
    HTR_CUDA(cudaGetLastError());
    return t;
}

ProjectedGram unfolding_refiner(Context& c, const DT& t, int mode, bool reduce) {
    return [&c, t, mode, reduce](const double* W, int64_t q) {
        const int64_t n = t.shape[static_cast<size_t>(mode)];
        DT B = mode_mul(c, t, mode, W, q, n, 1);  // W^T along `mode`
        return gram(c, B, mode, reduce);
    };
}

// ---------------------------------------------------------------------------
// input checks (bht.hpp:187-213) and tree plumbing
// ---------------------------------------------------------------------------

void check_batch_input(const Shape& ys, const DimensionTree& tree, const Shape* dims, const char* who) {
    const Index order = static_cast<Index>(ys.size());
    if (order != tree.dims() + 1)
        raise(HTR_ERR_INVALID_ARGUMENT, std::string(who) + ": tensor order " + std::to_string(order) +
                                            " does not match tree over " + std::to_string(tree.dims()) +
                                            " dims plus batch");
    if (order < 3) raise(HTR_ERR_INVALID_ARGUMENT, std::string(who) + ": need d >= 2 plus a batch axis");
    for (Index e : ys)
        if (e < 1) raise(HTR_ERR_INVALID_ARGUMENT, std::string(who) + ": extent < 1");
    if (dims) {
        for (Index k = 0; k < tree.dims(); ++k)
            if (ys[static_cast<size_t>(k)] != (*dims)[static_cast<size_t>(k)])
                raise(HTR_ERR_INVALID_ARGUMENT, std::string(who) + ": shape mismatch at mode " + std::to_string(k) +
                                                    ": " + std::to_string(ys[static_cast<size_t>(k)]) + " vs " +
                                                    std::to_string((*dims)[static_cast<size_t>(k)]));
    }
}

DimensionTree tree_from_nodes(const htr_node* nodes, int64_t n) {
    int32_t depth = -1;
    for (int64_t i = 0; i < n; ++i) depth = std::max(depth, nodes[i].layer);
    if (depth < 0) raise(HTR_ERR_INVALID_ARGUMENT, "DimensionTree: need a single root");
    std::vector<std::vector<TreeNode>> layers(static_cast<size_t>(depth) + 1);
    for (int64_t i = 0; i < n; ++i) {
        const htr_node& h = nodes[i];
        if (h.layer < 0) raise(HTR_ERR_INVALID_ARGUMENT, "DimensionTree: negative layer");
        auto& layer = layers[static_cast<size_t>(h.layer)];
        if (static_cast<int64_t>(layer.size()) <= h.pos) layer.resize(static_cast<size_t>(h.pos) + 1);
        TreeNode t;
        t.id = {h.layer, h.pos};
        t.kind = h.kind == HTR_KIND_ROOT ? NodeKind::Root : h.kind == HTR_KIND_TRANSFER ? NodeKind::Transfer : NodeKind::Leaf;
        t.leaf_dim = h.leaf_dim;
        if (h.succ0 >= 0) t.successors = {{h.layer + 1, h.succ0}, {h.layer + 1, h.succ1}};
        layer[static_cast<size_t>(h.pos)] = t;
    }
    try {
        return DimensionTree::from_layers(std::move(layers));
    } catch (const std::invalid_argument& e) {
        raise(HTR_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::out_of_range& e) {
        raise(HTR_ERR_OUT_OF_RANGE, e.what());
    }
}

void nodes_from_tree(const DimensionTree& t, std::vector<htr_node>& out) {
    out.clear();
    for (Index l = 0; l <= t.depth(); ++l)
        for (const TreeNode& n : t.layer(l)) {
            htr_node h;
            h.layer = static_cast<int32_t>(n.id.layer);
            h.pos = static_cast<int32_t>(n.id.pos);
            h.kind = n.kind == NodeKind::Root ? HTR_KIND_ROOT : n.kind == NodeKind::Transfer ? HTR_KIND_TRANSFER : HTR_KIND_LEAF;
            h.leaf_dim = static_cast<int32_t>(n.leaf_dim);
            h.succ0 = n.successors.empty() ? -1 : static_cast<int32_t>(n.successors[0].pos);
            h.succ1 = n.successors.empty() ? -1 : static_cast<int32_t>(n.successors[1].pos);
            out.push_back(h);
        }
}

namespace {

double effective_eps_rel(double eps_rel) {
    // bht.hpp:20-27
    if (!(eps_rel >= 0) || eps_rel >= 1.0) raise(HTR_ERR_INVALID_ARGUMENT, "relative tolerance must lie in [0, 1)");
    return eps_rel > 0 ? eps_rel : 1e-14;
}

double adaptive_budget(double eps_abs, double achieved_sq, Index remaining) {
    // bht.hpp:227-245
    if (remaining < 1) raise(HTR_ERR_INVALID_ARGUMENT, "adaptive_budget: no SVDs remaining");
    const double budget = eps_abs * eps_abs;
    double rem = budget - achieved_sq;
    if (rem < 0) {
        if (achieved_sq > budget * (1.0 + 1e-9) + 1e-300)
            raise(HTR_ERR_RUNTIME, "adaptive_budget: error budget exhausted (achieved^2 = " +
                                       std::to_string(achieved_sq) + " > eps_abs^2 = " + std::to_string(budget) + ")");
        rem = 0.0;
    }
    return std::sqrt(rem) / std::sqrt(static_cast<double>(remaining));
}

Index svds_below(const DimensionTree& t, Index l) {
    Index n = 0;
    for (Index k = 1; k < l; ++k) n += t.layer_size(k);
    return n;
}

Basis basis_of(const Rep& h, NodeId id) {
    const DT& c = h.core(id);
    if (h.tree.node(id).kind == NodeKind::Leaf) return {c.data(), c.shape[0], c.shape[1]};
    return {c.data(), c.shape[0] * c.shape[1], c.shape[2]};
}

/// Layer extent list with the batch last (bht.hpp:312-321); leaves already
/// projected by the fused kernel report their rank.
Shape layer_extents(const Rep& h, Index l, const RankMap& ranks, int64_t batch, bool leaves_projected) {
    Shape ext;
    for (const TreeNode& n : h.tree.layer(l)) {
        if (n.kind == NodeKind::Leaf)
            ext.push_back(leaves_projected ? ranks.at(n.id) : h.dims[static_cast<size_t>(n.leaf_dim)]);
        else
            ext.push_back(ranks.at(n.successors[0]) * ranks.at(n.successors[1]));
    }
    ext.push_back(batch);
    return ext;
}

namespace {

/// G_R = (I - U U^T) G (I - U U^T): the Gram of the residual
/// compute_residual(U, C) (ht_rise.hpp:31-38) without forming it.
void residual_gram(Context& c, DT& G, const Basis& U) {
    const int64_t a = U.alpha, r = U.r;
    DT X1 = c.tensor({r, a});
    {
        GemmDesc d;  // X1 = U^T G
        d.M = r; d.N1 = a; d.K1 = a;
        d.A = U.p; d.sam = a; d.sak1 = 1;
        d.B = G.data(); d.sbk1 = 1; d.sbn1 = a;
        d.C = X1.data(); d.scm = 1; d.scn1 = r;
        run_gemm(c, d);
    }
    {
        GemmDesc d;  // G -= U X1
        d.M = a; d.N1 = a; d.K1 = r;
        d.A = U.p; d.sam = 1; d.sak1 = a;
        d.B = X1.data(); d.sbk1 = 1; d.sbn1 = r;
        d.C = G.data(); d.scm = 1; d.scn1 = a;
        d.alpha = -1.0; d.beta = 1.0;
        run_gemm(c, d);
    }
    DT X2 = c.tensor({a, r});
    {
        GemmDesc d;  // X2 = G U
        d.M = a; d.N1 = r; d.K1 = a;
        d.A = G.data(); d.sam = 1; d.sak1 = a;
        d.B = U.p; d.sbk1 = 1; d.sbn1 = a;
        d.C = X2.data(); d.scm = 1; d.scn1 = a;
        run_gemm(c, d);
    }
    {
        GemmDesc d;  // G -= X2 U^T
        d.M = a; d.N1 = a; d.K1 = r;
        d.A = X2.data(); d.sam = 1; d.sak1 = a;
        d.B = U.p; d.sbk1 = a; d.sbn1 = 1;
        d.C = G.data(); d.scm = 1; d.scn1 = a;
        d.alpha = -1.0; d.beta = 1.0;
        run_gemm(c, d);
    }
}

}  // namespace

namespace {

/// K = X^T X (n x n) of a rows x n column-major matrix.
DT cols_gram(Context& c, const double* X, int64_t rows, int64_t n) {
    DT K = c.tensor({n, n});
    GemmDesc d;
    d.M = n; d.N1 = n; d.K1 = rows;
    d.A = X; d.sam = rows; d.sak1 = 1;
    d.B = X; d.sbk1 = 1; d.sbn1 = rows;
    d.C = K.data(); d.scm = 1; d.scn1 = n;
    run_gemm(c, d);
    return K;
}

/// Truncation of a rows x cols matrix X (rows > cols) through its column-side
/// Gram X^T X: the same singular values and rank rule (truncated_svd.hpp:
/// 53-100), left vectors U = X V_r Sigma_r^{-1}, re-orthonormalised by
/// CholeskyQR2. Small eigenvalues are re-measured through (X W)^T (X W).
Truncation truncate_cols_side(Context& c, const DT& X, int64_t rows, int64_t cols, double eps_abs, int64_t min_rank) {
    DT K = cols_gram(c, X.data(), rows, cols);
    ProjectedGram refine = [&c, X, rows, cols](const double* W, int64_t q) {
        DT Y = c.tensor({rows, q});
        GemmDesc d;  // Y = X W
        d.M = rows; d.N1 = q; d.K1 = cols;
        d.A = X.data(); d.sam = 1; d.sak1 = rows;
        d.B = W; d.sbk1 = 1; d.sbn1 = cols;
        d.C = Y.data(); d.scm = 1; d.scn1 = rows;
        run_gemm(c, d);
        return cols_gram(c, Y.data(), rows, q);
    };
    const Truncation tv = truncate_gram(c, K, cols, rows, eps_abs, min_rank, refine);
    Truncation t;
    t.rank = tv.rank;
    t.discarded = tv.discarded;
    t.sigma = tv.sigma;
    t.u = c.tensor({rows, t.rank});
    if (t.rank == 0) return t;
    const size_t r = static_cast<size_t>(t.rank);
    if (std::all_of(t.sigma.begin(), t.sigma.end(), [](double v) { return v == 0.0; })) {
        // zero matrix: the reference SVD's leading identity columns
        std::vector<double> e(static_cast<size_t>(rows) * r, 0.0);
        for (size_t i = 0; i < r; ++i) e[i + static_cast<size_t>(rows) * i] = 1.0;
        HTR_CUDA(cudaMemcpyAsync(t.u.data(), e.data(), sizeof(double) * e.size(), cudaMemcpyHostToDevice, c.s));
        HTR_CUDA(cudaStreamSynchronize(c.s));
        return t;
    }
    std::vector<double> v(static_cast<size_t>(cols) * r);
    c.fetch(tv.u.data(), static_cast<int64_t>(v.size()), v.data());
    for (size_t j = 0; j < r; ++j) {
        const double inv = t.sigma[j] > 0.0 ? 1.0 / t.sigma[j] : 0.0;
        for (int64_t i = 0; i < cols; ++i) v[static_cast<size_t>(i) + static_cast<size_t>(cols) * j] *= inv;
    }
    DT Vs = c.tensor({cols, t.rank});
    HTR_CUDA(cudaMemcpyAsync(Vs.data(), v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, c.s));
    {
        GemmDesc d;  // U = X V_r Sigma_r^{-1}
        d.M = rows; d.N1 = t.rank; d.K1 = cols;
        d.A = X.data(); d.sam = 1; d.sak1 = rows;
        d.B = Vs.data(); d.sbk1 = 1; d.sbn1 = cols;
        d.C = t.u.data(); d.scm = 1; d.scn1 = rows;
        run_gemm(c, d);
    }
    BufPtr info = c.alloc(4);
    BufPtr work = c.alloc(t.rank * t.rank + 16);
    launch_orthonormalize_new(nullptr, rows, 0, t.u.data(), t.rank, info->p, work->p, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    HTR_CUDA(cudaStreamSynchronize(c.s));  // v is pageable host memory
    return t;
}

}  // namespace

}  // namespace

namespace {
/// The old-basis (residual) truncation's set-up on the unfolding Gram G:
/// G <- (I - U U^T) G (I - U U^T), its noise scale (tr of the unprojected
/// Gram) and the refiner that re-measures small eigenvalues on the residual.
std::pair<double, ProjectedGram> residual_setup(Context& c, const DT& t, int mode, const Basis U, bool reduce, DT& G) {
    const int64_t rows = t.shape[static_cast<size_t>(mode)];
    // the residual Gram is formed by subtraction: its eigenvalues carry
    // rounding noise on the scale of the unprojected Gram (its trace)
    std::vector<double> diag(static_cast<size_t>(rows));
    HTR_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double), G.data(), sizeof(double) * static_cast<size_t>(rows + 1),
                               sizeof(double), static_cast<size_t>(rows), cudaMemcpyDeviceToHost, c.s));
    residual_gram(c, G, U);
    HTR_CUDA(cudaStreamSynchronize(c.s));
    double gtrace = 0.0;
    for (double v : diag) gtrace += v;
    // refinement measures the residual R = (I - U U^T) C directly:
    // W^T R = ((I - U U^T) W)^T C
    ProjectedGram refine = [&c, t, mode, U, reduce](const double* W, int64_t q) {
        DT T = c.tensor({U.r, q});
        {
            GemmDesc d;  // T = U^T W
            d.M = U.r; d.N1 = q; d.K1 = U.alpha;
            d.A = U.p; d.sam = U.alpha; d.sak1 = 1;
            d.B = W; d.sbk1 = 1; d.sbn1 = U.alpha;
            d.C = T.data(); d.scm = 1; d.scn1 = U.r;
            run_gemm(c, d);
        }
        DT Wp = c.tensor({U.alpha, q});
        HTR_CUDA(cudaMemcpyAsync(Wp.data(), W, sizeof(double) * static_cast<size_t>(U.alpha * q),
                                 cudaMemcpyDeviceToDevice, c.s));
        {
            GemmDesc d;  // Wp -= U T
            d.M = U.alpha; d.N1 = q; d.K1 = U.r;
            d.A = U.p; d.sam = 1; d.sak1 = U.alpha;
            d.B = T.data(); d.sbk1 = 1; d.sbn1 = U.r;
            d.C = Wp.data(); d.scm = 1; d.scn1 = U.alpha;
            d.alpha = -1.0; d.beta = 1.0;
            run_gemm(c, d);
        }
        DT B = mode_mul(c, t, mode, Wp.data(), q, U.alpha, 1);
        return gram(c, B, mode, reduce);
    };
    return {gtrace, refine};
}
}  // namespace

namespace {
/// Full-rank certificate of a Gram (the shortcut for the Grams that need the
/// cluster eigensolver, n > 160, tens of ms; a failed test costs ~2 ms):
/// Cholesky of G - (eps^2 + 1e-12 tr G) I on `st`; margin 1e-12 tr(G) >>
/// n u ||G||. The trace is read on the context stream first.
struct PosdefProbe {
    bool launched = false;
    BufPtr work, flag;
    std::vector<BufPtr> gemm_ws;  // trailing-update workspaces, live until finish
};
PosdefProbe posdef_launch(Context& c, const DT& G, int64_t rows, double eps_abs, cudaStream_t st) {
    PosdefProbe pr;
    std::vector<double> diag(static_cast<size_t>(rows));
    HTR_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double), G.data(), sizeof(double) * static_cast<size_t>(rows + 1),
                               sizeof(double), static_cast<size_t>(rows), cudaMemcpyDeviceToHost, c.s));
    HTR_CUDA(cudaStreamSynchronize(c.s));
    double tr = 0.0;
    for (double v : diag) tr += v;
    if (!(tr > 0.0 && std::isfinite(tr))) return pr;
    pr.work = c.alloc(rows * rows);
    pr.flag = c.alloc(4);
    HTR_CUDA(cudaMemsetAsync(pr.flag->p, 0, 4 * sizeof(double), c.s));
    // blocked right-looking Cholesky: 32-column panels (one CTA each), the
    // trailing updates A22 -= P P^T on the DMMA GEMM engine
    const int64_t n = rows;
    std::vector<GemmDesc> upd;
    for (int64_t kb = 0; kb + kCholPanel < n; kb += kCholPanel) {
        const int64_t m = n - kb - kCholPanel;
        double* P = pr.work->p + (kb + kCholPanel) + n * kb;
        GemmDesc d;
        d.M = m; d.N1 = m; d.K1 = kCholPanel;
        d.A = P; d.sam = 1; d.sak1 = n;
        d.B = P; d.sbk1 = n; d.sbn1 = 1;
        d.C = pr.work->p + (kb + kCholPanel) + n * (kb + kCholPanel); d.scm = 1; d.scn1 = n;
        d.alpha = -1.0; d.beta = 1.0;
        const int64_t ws = gemm_workspace_doubles(d, c.num_sms);
        pr.gemm_ws.push_back(ws > 0 ? c.alloc(ws) : nullptr);
        upd.push_back(d);
    }
    if (st != c.s) {  // the buffers, workspaces and G are ordered on the context stream
        HTR_CUDA(cudaEventRecord(c.aux_ev, c.s));
        HTR_CUDA(cudaStreamWaitEvent(st, c.aux_ev, 0));
    }
    launch_chol_prepare(G.data(), n, eps_abs * eps_abs + 1e-12 * tr, pr.work->p, pr.flag->p, st, &c.launches);
    for (int64_t kb = 0, p = 0; kb < n; kb += kCholPanel, ++p) {
        launch_chol_panel(pr.work->p, n, kb, std::min(kCholPanel, n - kb), pr.flag->p, st, &c.launches);
        if (kb + kCholPanel < n) {
            const BufPtr& w = pr.gemm_ws[static_cast<size_t>(p)];
            launch_gemm(upd[static_cast<size_t>(p)], w ? w->p : nullptr, c.num_sms, st, &c.launches);
        }
    }
    HTR_CUDA(cudaGetLastError());
    pr.launched = true;
    return pr;
}
/// Reads the certificate (synchronising `st`); on success *out is the
/// identity basis of the full space.
bool posdef_finish(Context& c, PosdefProbe& pr, int64_t rows, cudaStream_t st, Truncation* out) {
    if (!pr.launched) return false;
    double f = 0.0;
    HTR_CUDA(cudaMemcpyAsync(&f, pr.flag->p, sizeof(double), cudaMemcpyDeviceToHost, st));
    HTR_CUDA(cudaStreamSynchronize(st));
    if (f != 1.0) return false;
    out->rank = rows;
    out->discarded = 0.0;
    out->u = c.tensor({rows, rows});
    // take_columns with a zero-input flag (flag[2] == 0) writes identity columns
    launch_take_columns(nullptr, rows, rows, out->u.data(), pr.flag->p, c.s, &c.launches);
    out->u.buf->identity = true;
    HTR_CUDA(cudaGetLastError());
    return true;
}
}  // namespace

Truncation truncate_mode(Context& c, const DT& t, int mode, const Basis* old, double eps_abs, int64_t min_rank,
                         int64_t cols_global, bool sharded, bool any_basis_when_full) {
    const int64_t rows = t.shape[static_cast<size_t>(mode)];
    const int64_t cols_local = t.size() / rows;
    const bool reduce = sharded && c.sharded();
    if (!reduce && rows > kColumnSideRows && cols_local < rows) {
        // tall unfolding on one rank: decompose the smaller, column-side Gram
        int64_t inner = 1, outer = 1;
        for (int k = 0; k < mode; ++k) inner *= t.shape[static_cast<size_t>(k)];
        for (size_t k = static_cast<size_t>(mode) + 1; k < t.shape.size(); ++k) outer *= t.shape[k];
        DT X = c.tensor({rows, cols_local});
        launch_unfold(t.data(), inner, rows, outer, X.data(), c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        if (old && old->r > 0) {
            // explicit residual X <- (I - U U^T) X (compute_residual, ht_rise.hpp:31-38)
            DT T = c.tensor({old->r, cols_local});
            GemmDesc d;  // T = U^T X
            d.M = old->r; d.N1 = cols_local; d.K1 = rows;
            d.A = old->p; d.sam = rows; d.sak1 = 1;
            d.B = X.data(); d.sbk1 = 1; d.sbn1 = rows;
            d.C = T.data(); d.scm = 1; d.scn1 = old->r;
            run_gemm(c, d);
            GemmDesc e;  // X -= U T
            e.M = rows; e.N1 = cols_local; e.K1 = old->r;
            e.A = old->p; e.sam = 1; e.sak1 = rows;
            e.B = T.data(); e.sbk1 = 1; e.sbn1 = old->r;
            e.C = X.data(); e.scm = 1; e.scn1 = rows;
            e.alpha = -1.0; e.beta = 1.0;
            run_gemm(c, e);
        }
        return truncate_cols_side(c, X, rows, cols_local, eps_abs, min_rank);
    }
    if (reduce && rows > kColumnSideRows && cols_global < rows) {
        // tall unfolding, batch-sharded: the column-side Gram needs every
        // column, so each rank gathers the whole unfolding -- its own columns
        // are one contiguous block (the batch axis is the slowest) -- through
        // an all-reduce of a zero-initialised buffer and truncates it like a
        // single rank; every rank computes the same bits
        int64_t inner = 1, outer = 1;
        for (int k = 0; k < mode; ++k) inner *= t.shape[static_cast<size_t>(k)];
        for (size_t k = static_cast<size_t>(mode) + 1; k < t.shape.size(); ++k) outer *= t.shape[k];
        const int64_t batch = t.shape.back();
        const int64_t per_sample = inner * (outer / batch);  // unfolding columns per sample
        BufPtr counts = c.alloc(c.nranks);
        HTR_CUDA(cudaMemsetAsync(counts->p, 0, sizeof(double) * static_cast<size_t>(c.nranks), c.s));
        c.h_sc[0] = static_cast<double>(batch);
        HTR_CUDA(cudaMemcpyAsync(counts->p + c.rank, c.h_sc, sizeof(double), cudaMemcpyHostToDevice, c.s));
        c.allreduce(counts->p, c.nranks);
        std::vector<double> cnt(static_cast<size_t>(c.nranks));
        c.fetch(counts->p, c.nranks, cnt.data());
        int64_t s_off = 0, s_all = 0;
        for (int r = 0; r < c.nranks; ++r) {
            if (r < c.rank) s_off += static_cast<int64_t>(std::llround(cnt[static_cast<size_t>(r)]));
            s_all += static_cast<int64_t>(std::llround(cnt[static_cast<size_t>(r)]));
        }
        const int64_t cols_all = per_sample * s_all;
        DT X = c.tensor({rows, cols_all});
        HTR_CUDA(cudaMemsetAsync(X.data(), 0, sizeof(double) * static_cast<size_t>(rows * cols_all), c.s));
        launch_unfold(t.data(), inner, rows, outer, X.data() + rows * per_sample * s_off, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        c.allreduce(X.data(), rows * cols_all);
        if (old && old->r > 0) {
            DT T = c.tensor({old->r, cols_all});
            GemmDesc d;  // T = U^T X
            d.M = old->r; d.N1 = cols_all; d.K1 = rows;
            d.A = old->p; d.sam = rows; d.sak1 = 1;
            d.B = X.data(); d.sbk1 = 1; d.sbn1 = rows;
            d.C = T.data(); d.scm = 1; d.scn1 = old->r;
            run_gemm(c, d);
            GemmDesc e;  // X -= U T
            e.M = rows; e.N1 = cols_all; e.K1 = old->r;
            e.A = old->p; e.sam = 1; e.sak1 = rows;
            e.B = T.data(); e.sbk1 = 1; e.sbn1 = old->r;
            e.C = X.data(); e.scm = 1; e.scn1 = rows;
            e.alpha = -1.0; e.beta = 1.0;
            run_gemm(c, e);
        }
        return truncate_cols_side(c, X, rows, cols_all, eps_abs, min_rank);
    }
    DT G = gram(c, t, mode, reduce);
    if (!old && any_basis_when_full && rows > 160 && rows <= cols_global && tridiag_supported(rows)) {
        PosdefProbe probe = posdef_launch(c, G, rows, eps_abs, c.s);
        Truncation full;
        if (posdef_finish(c, probe, rows, c.s, &full)) return full;
    }
    if (!old) return truncate_gram(c, G, rows, cols_global, eps_abs, min_rank, unfolding_refiner(c, t, mode, reduce));
    double gtrace = 0.0;
    ProjectedGram refine;
    std::tie(gtrace, refine) = residual_setup(c, t, mode, *old, reduce, G);
    return truncate_gram(c, G, rows, cols_global, eps_abs, min_rank, refine, gtrace);
}

std::vector<Truncation> truncate_modes(Context& c, const DT& t, const std::vector<int>& modes, double eps_abs,
                                       int64_t min_rank, const std::vector<int64_t>& cols_global, bool sharded,
                                       bool any_basis_when_full, const std::vector<Basis>* olds) {
    // the unprojected truncations (no old basis) that take the plain Gram ->
    // one-CTA eigensolver route are batched: their Grams first, then one
    // launch solving all of them side by side (bit-identical to one by one)
    const bool reduce = sharded && c.sharded();
    std::vector<char> batch(modes.size(), 0), pdef(modes.size(), 0);
    int nb = 0, npd = 0;
    for (size_t i = 0; i < modes.size(); ++i) {
        const int64_t rows = t.shape[static_cast<size_t>(modes[i])];
        const int64_t cols_local = t.size() / rows;
        const bool column_side = rows > kColumnSideRows && (reduce ? cols_global[i] < rows : cols_local < rows);
        const bool posdef =
            !olds && any_basis_when_full && rows > 160 && rows <= cols_global[i] && tridiag_supported(rows);
        batch[i] = !column_side && !posdef && (c.tridiag ? tridiag_supported(rows) : jacobi_batchable(rows));
        pdef[i] = !column_side && posdef;
        nb += batch[i];
        npd += pdef[i];
    }
    std::vector<Truncation> out(modes.size());
    auto old_of = [&](size_t i) { return olds ? &(*olds)[i] : nullptr; };
    if (nb < 2 && !(nb == 1 && npd > 0)) {
        for (size_t i = 0; i < modes.size(); ++i)
            out[i] = truncate_mode(c, t, modes[i], old_of(i), eps_abs, min_rank, cols_global[i], sharded,
                                   any_basis_when_full);
        return out;
    }
    // full-rank certificates run on the auxiliary stream, beside the batched
    // eigensolve on the context stream (c5's layer 1: the 400-row transfer
    // Gram's Cholesky next to the 128-row leaf solve)
    std::vector<DT> pgrams(modes.size());
    std::vector<PosdefProbe> probes(modes.size());
    for (size_t i = 0; i < modes.size(); ++i) {
        if (!pdef[i]) continue;
        pgrams[i] = gram(c, t, modes[i], reduce);
        probes[i] = posdef_launch(c, pgrams[i], t.shape[static_cast<size_t>(modes[i])], eps_abs, c.s_aux);
    }
    std::vector<ProjectedGram> refiners;
    std::vector<double> noise;
    std::vector<DT> grams;
    std::vector<BufPtr> lams, vs;
    std::vector<const double*> gp;
    std::vector<int64_t> ns;
    std::vector<double*> lp, vp;
    for (size_t i = 0; i < modes.size(); ++i) {
        if (!batch[i]) continue;
        const int64_t rows = t.shape[static_cast<size_t>(modes[i])];
        grams.push_back(gram(c, t, modes[i], reduce));
        if (olds) {
            double gtrace = 0.0;
            ProjectedGram refine;
            std::tie(gtrace, refine) = residual_setup(c, t, modes[i], (*olds)[i], reduce, grams.back());
            refiners.push_back(refine);
            noise.push_back(gtrace);
        } else {
            refiners.push_back(unfolding_refiner(c, t, modes[i], reduce));
            noise.push_back(0.0);
        }
        lams.push_back(c.alloc(rows));
        vs.push_back(c.tridiag ? nullptr : c.alloc(rows * rows));
        gp.push_back(grams.back().data());
        ns.push_back(rows);
        lp.push_back(lams.back()->p);
        vp.push_back(vs.back() ? vs.back()->p : nullptr);
    }
    std::vector<TriSolve> tris;
    if (c.tridiag) {
        std::vector<double*> wp;
        for (size_t j = 0; j < ns.size(); ++j) {
            tris.push_back(TriSolve{lams[j], c.alloc(tridiag_workspace_doubles(ns[j])), ns[j]});
            wp.push_back(tris.back().W->p);
        }
        launch_tridiag_eigvals(gp.data(), ns.data(), lp.data(), wp.data(), nb, c.s, &c.launches);
    } else {
        launch_jacobi_eig_batch(gp.data(), ns.data(), lp.data(), vp.data(), nb, c.s, &c.launches);
    }
    HTR_CUDA(cudaGetLastError());
    std::vector<Truncation> tri_out;
    if (c.tridiag) {
        std::vector<int64_t> bcols;
        for (size_t i = 0; i < modes.size(); ++i)
            if (batch[i]) bcols.push_back(cols_global[i]);
        tri_out = finish_tri_batch(c, tris, grams, ns, bcols, eps_abs, min_rank, refiners, noise);
    }
    for (size_t i = 0, j = 0; i < modes.size(); ++i) {
        if (batch[i]) {
            out[i] = c.tridiag ? std::move(tri_out[j])
                               : truncate_eig(c, lams[j], vs[j], ns[j], cols_global[i], eps_abs, min_rank,
                                              refiners[j], noise[j]);
            ++j;
        } else if (pdef[i]) {
            const int64_t rows = t.shape[static_cast<size_t>(modes[i])];
            if (!posdef_finish(c, probes[i], rows, c.s_aux, &out[i]))
                out[i] = truncate_gram(c, pgrams[i], rows, cols_global[i], eps_abs, min_rank,
                                       unfolding_refiner(c, t, modes[i], reduce));
        } else {
            out[i] = truncate_mode(c, t, modes[i], old_of(i), eps_abs, min_rank, cols_global[i], sharded,
                                   any_basis_when_full);
        }
    }
    return out;
}

namespace {

/// t x_mode U^T. With energy_slot the explicit residual energy of the step
/// is added there; with ysq_slot ||t||^2 is written there when the streaming
/// kernel runs (*ysq_done reports whether it did).
DT project(Context& c, const DT& t, int mode, const Basis& b, double* energy_slot, double* ysq_slot = nullptr,
           bool* ysq_done = nullptr, const DT* dst = nullptr) {
    if (b.alpha != t.shape[static_cast<size_t>(mode)])
        raise(HTR_ERR_INVALID_ARGUMENT, "mode_multiply: factor/extent mismatch");
    const Split sp = split_at(t.shape, mode);
    if (ysq_done) *ysq_done = false;
    if ((energy_slot || ysq_slot) && sp.J <= 16 && b.r <= 16 && sp.I * sp.O >= 4096) {
        // streaming projection with the explicit residual energy and/or the
        // input's squared norm fused in
        Shape os = t.shape;
        os[static_cast<size_t>(mode)] = b.r;
        DT coeff = c.tensor(os);
        BufPtr parts = energy_slot ? c.alloc(8 * c.num_sms) : nullptr;
        BufPtr yparts = ysq_slot ? c.alloc(8 * c.num_sms) : nullptr;
        const int nb = launch_mode_small(t.data(), sp.I, sp.J, sp.O, b.p, b.r, b.alpha, 1, coeff.data(),
                                         parts ? parts->p : nullptr, yparts ? yparts->p : nullptr, c.num_sms, c.s,
                                         &c.launches);
        if (nb > 0) {
            if (parts) launch_sum_partials(parts->p, nb, energy_slot, c.s, &c.launches);
            if (yparts) launch_sum_partials(yparts->p, nb, ysq_slot, c.s, &c.launches);
            HTR_CUDA(cudaGetLastError());
            if (ysq_done) *ysq_done = ysq_slot != nullptr;
            return coeff;
        }
    }
    if (dst && !energy_slot) {
        // straight into caller memory (a skip's latent into the root store's
        // next slices): the returned view is the caller's, so a later root
        // append sees it in place
        Shape os = t.shape;
        os[static_cast<size_t>(mode)] = b.r;
        if (dst->shape == os) {
            mode_mul(c, t, mode, b.p, b.r, b.alpha, 1, dst->data());
            return *dst;
        }
    }
    DT coeff = mode_mul(c, t, mode, b.p, b.r, b.alpha, 1);  // U^T
    if (energy_slot) residual_energy(c, t, mode, b.p, b.r, coeff, energy_slot);
    return coeff;
}

/// t x_mode U1^T x_(mode+1) U2^T in one read of t (k_proj2.cu) when the
/// shapes fit the fused kernel; false (nothing launched) otherwise.
bool project_pair(Context& c, const DT& t, int mode, const Basis& b1, const Basis& b2, DT* out) {
    if (!c.fused || mode + 2 > static_cast<int>(t.shape.size())) return false;
    const Split sp = split_at(t.shape, mode);  // [I, J, O]
    Proj2Args a;
    a.Y = t.data();
    a.n0 = sp.I;
    a.n1 = sp.J;
    a.n2 = t.shape[static_cast<size_t>(mode) + 1];
    a.S = sp.O / a.n2;
    a.U1 = b1.p;
    a.U2 = b2.p;
    a.r1 = static_cast<int>(b1.r);
    a.r2 = static_cast<int>(b2.r);
    if (b1.alpha != a.n1 || b2.alpha != a.n2 || !proj2_supported(a)) return false;
    Shape os = t.shape;
    os[static_cast<size_t>(mode)] = b1.r;
    os[static_cast<size_t>(mode) + 1] = b2.r;
    DT o = c.tensor(os);
    a.C = o.data();
    if (launch_proj2(a, c.s, &c.launches) < 0) return false;
    HTR_CUDA(cudaGetLastError());
    *out = o;
    return true;
}

/// The projections of a layer's leaves in layer order (bht.hpp:290-293,
/// ht_rise.hpp:160-162); two leaves over adjacent modes go through the fused
/// pair kernel when it applies.
DT project_leaves(Context& c, DT cur, const std::vector<TreeNode>& leaves, const std::vector<Basis>& bases) {
    for (size_t i = 0; i < leaves.size();) {
        const int mode = static_cast<int>(leaves[i].leaf_dim);
        DT pr;
        if (i + 1 < leaves.size() && leaves[i + 1].leaf_dim == leaves[i].leaf_dim + 1 &&
            project_pair(c, cur, mode, bases[i], bases[i + 1], &pr)) {
            cur = pr;
            i += 2;
            continue;
        }
        cur = project(c, cur, mode, bases[i], nullptr);
        ++i;
    }
    return cur;
}

int64_t global_batch(Context& c, int64_t local) {
    if (!c.sharded()) return local;
    c.h_sc[0] = static_cast<double>(local);
    HTR_CUDA(cudaMemcpyAsync(c.d_sc->p + 8, c.h_sc, sizeof(double), cudaMemcpyHostToDevice, c.s));
    c.allreduce(c.d_sc->p + 8, 1);
    double g = 0.0;
    c.fetch(c.d_sc->p + 8, 1, &g);
    return static_cast<int64_t>(std::llround(g));
}

std::shared_ptr<RootStore> new_root(Context& c, int64_t r11, int64_t r12, int64_t cap) {
    auto rs = std::make_shared<RootStore>();
    rs->r11 = r11;
    rs->r12 = r12;
    rs->cap = std::max<int64_t>(cap, 1);
    rs->buf = c.alloc(r11 * r12 * rs->cap);
    rs->committed = 0;
    return rs;
}

}  // namespace

// ---------------------------------------------------------------------------
// BHT-l2r (bht.hpp:251-350)
// ---------------------------------------------------------------------------

BuildOut bht_l2r(Context& c, const DT& y, const DimensionTree& tree, double eps_rel, bool adaptive) {
    check_batch_input(y.shape, tree, nullptr, "bht_l2r");
    const Index d = tree.dims(), p = tree.depth();
    const int64_t batch = y.shape[static_cast<size_t>(d)];
    const int64_t gbatch = global_batch(c, batch);
    double ysq = 0.0;
    bool have_ysq = false;
    {
        // ||y||^2 = trace of the first leaf's mode Gram, which its truncation
        // needs anyway: one pass over y less than a separate norm scan
        const int mode = static_cast<int>(tree.layer(p)[0].leaf_dim);
        const int64_t rows = y.shape[static_cast<size_t>(mode)];
        const bool column_side = !c.sharded() && rows > kColumnSideRows && y.size() / rows < rows;
        if (!column_side) {
            DT G = gram(c, y, mode, true);
            std::vector<double> diag(static_cast<size_t>(rows));
            HTR_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double), G.data(), sizeof(double) * static_cast<size_t>(rows + 1),
                                       sizeof(double), static_cast<size_t>(rows), cudaMemcpyDeviceToHost, c.s));
            HTR_CUDA(cudaStreamSynchronize(c.s));
            for (double v : diag) ysq += v;
            if (std::isfinite(ysq)) {
                c.gram_hint = Context::GramHint{y.data(), mode, y.shape, G};
                have_ysq = true;
            }
        }
    }
    if (!have_ysq) {  // (also distinguishes non-finite input from overflow)
        bool bad = false;
        norm_sq(c, y.data(), y.size(), &ysq, &bad);
        if (bad) raise(HTR_ERR_INVALID_ARGUMENT, "bht_l2r: non-finite input");
    }
    const double norm_y = std::sqrt(ysq);
    const double eps_abs = effective_eps_rel(eps_rel) * norm_y;

    BuildOut out;
    std::memset(&out.report, 0, sizeof(out.report));
    htr_build_report& rep = out.report;
    rep.eps_nw_initial = eps_abs / std::sqrt(static_cast<double>(2 * d - 2));
    rep.layer_norms[rep.n_layer_norms++] = norm_y;

    auto h = std::make_shared<Rep>();
    h->st = c.st;
    h->tree = tree;
    h->dims = Shape(y.shape.begin(), y.shape.end() - 1);
    h->cores.resize(static_cast<size_t>(p) + 1);
    for (Index l = 0; l <= p; ++l) h->cores[static_cast<size_t>(l)].resize(static_cast<size_t>(tree.layer_size(l)));
    h->eps_rel = eps_rel;

    auto record = [&](NodeId id, int64_t rank, double disc) {
        if (rep.n_records < HTR_MAX_NODES) {
            rep.rec_layer[rep.n_records] = static_cast<int32_t>(id.layer);
            rep.rec_pos[rep.n_records] = static_cast<int32_t>(id.pos);
            rep.rec_rank[rep.n_records] = rank;
            rep.rec_discarded[rep.n_records] = disc;
            ++rep.n_records;
        }
    };
    auto push_norm = [&](const DT& t) {
        double s = 0.0;
        norm_sq(c, t.data(), t.size(), &s, nullptr);
        if (rep.n_layer_norms < HTR_MAX_LAYERS) rep.layer_norms[rep.n_layer_norms++] = std::sqrt(s);
        return std::sqrt(s);
    };

    double eps_nw = rep.eps_nw_initial;
    DT cur = y;
    const double col_scale = static_cast<double>(gbatch) / static_cast<double>(batch);
    auto cols_of = [&](const DT& t, int mode) {
        const int64_t J = t.shape[static_cast<size_t>(mode)];
        return static_cast<int64_t>(std::llround(static_cast<double>(t.size() / J) * col_scale));
    };

    // deepest layer: plain HOSVD of y over all leaves, then sequential projections
    std::vector<int> leaf_modes;
    std::vector<int64_t> leaf_cols;
    for (const TreeNode& n : tree.layer(p)) {
        leaf_modes.push_back(static_cast<int>(n.leaf_dim));
        leaf_cols.push_back(cols_of(cur, leaf_modes.back()));
    }
    std::vector<Truncation> bases = truncate_modes(c, cur, leaf_modes, eps_nw, 1, leaf_cols, true, true);
    RankMap ranks;
    for (size_t i = 0; i < bases.size(); ++i) {
        const TreeNode& n = tree.layer(p)[i];
        DT core = bases[i].u;
        h->cores[static_cast<size_t>(p)][i] = core;
        ranks[n.id] = bases[i].rank;
        record(n.id, bases[i].rank, bases[i].discarded);
    }
    {
        std::vector<Basis> lb;
        for (const Truncation& b : bases) lb.push_back({b.u.data(), b.u.shape[0], b.rank});
        cur = project_leaves(c, cur, tree.layer(p), lb);
    }
    push_norm(cur);

    for (Index l = p - 1; l >= 1; --l) {
        if (adaptive) {
            const double cn = rep.layer_norms[rep.n_layer_norms - 1];
            eps_nw = adaptive_budget(eps_abs, std::max(0.0, ysq - cn * cn), svds_below(tree, l + 1));
        }
        cur.shape = layer_extents(*h, l, ranks, batch, false);
        std::vector<int> lmodes;
        std::vector<int64_t> lcols;
        for (Index j = 0; j < tree.layer_size(l); ++j) {
            lmodes.push_back(static_cast<int>(j));
            lcols.push_back(cols_of(cur, static_cast<int>(j)));
        }
        std::vector<Truncation> lb = truncate_modes(c, cur, lmodes, eps_nw, 1, lcols, true, true);
        for (Index j = 0; j < tree.layer_size(l); ++j) {
            const TreeNode& n = tree.layer(l)[static_cast<size_t>(j)];
            Truncation& b = lb[static_cast<size_t>(j)];
            DT core = b.u;
            if (n.kind != NodeKind::Leaf) core.shape = {ranks[n.successors[0]], ranks[n.successors[1]], b.rank};
            h->cores[static_cast<size_t>(l)][static_cast<size_t>(j)] = core;
            ranks[n.id] = b.rank;
            record(n.id, b.rank, b.discarded);
        }
        for (Index j = 0; j < tree.layer_size(l); ++j) {
            const Truncation& b = lb[static_cast<size_t>(j)];
            cur = project(c, cur, static_cast<int>(j), {b.u.data(), b.u.shape[0], b.rank}, nullptr);
        }
        push_norm(cur);
    }

    const TreeNode& rootn = tree.node({0, 0});
    const int64_t r11 = ranks[rootn.successors[0]], r12 = ranks[rootn.successors[1]];
    h->root = new_root(c, r11, r12, batch);
    HTR_CUDA(cudaMemcpyAsync(h->root->buf->p, cur.data(), sizeof(double) * static_cast<size_t>(r11 * r12 * batch),
                             cudaMemcpyDeviceToDevice, c.s));
    h->root->committed = batch;
    h->acc = batch;
    h->acc_global = gbatch;
    measure_defect(c, *h);
    out.rep = h;
    return out;
}

// ---------------------------------------------------------------------------
// encode (bht.hpp:373-401)
// ---------------------------------------------------------------------------

namespace {

struct Tree3 {
    NodeId leaf_of[3];
    int r0 = 0, r1 = 0, r2 = 0, rt = 0;
    bool tree_123 = false;  // (1,(2,3)): layer 1 = [leaf d0, transfer(d1,d2)]
};

Tree3 tree3_ranks(const Rep& h, const RankMap& ranks) {
    const DimensionTree& tree = h.tree;
    Tree3 t;
    for (Index l = 1; l <= tree.depth(); ++l)
        for (const TreeNode& n : tree.layer(l))
            if (n.kind == NodeKind::Leaf) t.leaf_of[n.leaf_dim] = n.id;
    t.r0 = static_cast<int>(ranks.at(t.leaf_of[0]));
    t.r1 = static_cast<int>(ranks.at(t.leaf_of[1]));
    t.r2 = static_cast<int>(ranks.at(t.leaf_of[2]));
    t.tree_123 = tree.depth() == 2 && tree.layer(1)[0].kind == NodeKind::Leaf &&
                 tree.layer(1)[1].kind == NodeKind::Transfer;
    t.rt = t.tree_123 ? static_cast<int>(ranks.at(NodeId{1, 1})) : 0;
    return t;
}

}  // namespace

bool launch_skip_encode3(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc, DT* latent,
                         cudaEvent_t ev0, cudaEvent_t ev1, double* host_out) {
    if (h.tree.dims() != 3 || h.tree.depth() != 2) return false;
    const Tree3 t = tree3_ranks(h, h.ranks());
    const int64_t batch = y.shape[3];
    if (!t.tree_123 || !tail3_supported(t.r0, t.r1, t.r2, t.rt, y.shape[2]) ||
        !fused3_supported(y.shape[0], y.shape[1], y.shape[2], t.r0, t.r1, t.r2))
        return false;
    Fused3Args fa;
    fa.Y = y.data();
    fa.n2 = y.shape[2];
    fa.S = batch;
    fa.U0 = h.core(t.leaf_of[0]).data();
    fa.U1 = h.core(t.leaf_of[1]).data();
    fa.U2 = h.core(t.leaf_of[2]).data();
    fa.r0 = t.r0;
    fa.r1 = t.r1;
    fa.r2 = t.r2;
    fa.slab_gemm = false;
    const int64_t ws = fused3_workspace_doubles(y.shape[0], y.shape[1], fa.n2, batch, t.r0, t.r1, t.r2, c.num_sms);
    BufPtr w = c.alloc(ws);  // freed stream-ordered after the kernels below
    fa.wslab = w->p;
    fa.ysq_partials = w->p + fa.n2 * batch * static_cast<int64_t>(t.r0) * t.r1;
    if (ev0) HTR_CUDA(cudaEventRecord(ev0, c.s));
    const int grid = launch_fused3(y.shape[0], y.shape[1], fa, c.num_sms, c.s, &c.launches);
    if (ev1) HTR_CUDA(cudaEventRecord(ev1, c.s));
    HTR_CUDA(cudaGetLastError());
    if (grid <= 0) return false;  // no tensor map for this pointer: nothing was launched
    Tail3Args ta;
    ta.wslab = fa.wslab;
    ta.U2 = fa.U2;
    const DT& Bcore = h.core(NodeId{1, 1});
    ta.B = Bcore.data();
    ta.identity_transfer = Bcore.buf->identity && Bcore.offset == 0 && t.rt == t.r1 * t.r2;
    ta.r0 = t.r0;
    ta.r1 = t.r1;
    ta.r2 = t.r2;
    ta.rt = t.rt;
    ta.n2 = fa.n2;
    ta.S = batch;
    DT lat;
    if (latent_target && latent_target->shape == Shape{t.r0, t.rt, batch}) {
        lat = *latent_target;
    } else {
        lat = c.tensor({t.r0, t.rt, batch});
    }
    ta.latent = lat.data();
    ta.variant = c.tail_kernel;
    ta.num_sms = c.num_sms;
    BufPtr lsq = c.alloc(tail3_latsq_entries(batch, c.num_sms));  // per-CTA partials
    ta.latsq = lsq->p;
    ta.ysq_partials = fa.ysq_partials;
    ta.n_ysq = grid;
    ta.out = sc;
    ta.host_out = host_out;
    ta.ticket = c.d_ticket;
    launch_tail3(ta, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    *latent = lat;
    return true;
}

bool launch_skip_encode8(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc, DT* latent,
                         cudaEvent_t ev0, cudaEvent_t ev1, double* host_out) {
    const DimensionTree& tree = h.tree;
    if (tree.dims() != 8 || tree.depth() != 3) return false;
    for (int k = 0; k < 8; ++k)
        if (y.shape[static_cast<size_t>(k)] != 8) return false;
    const RankMap ranks = h.ranks();
    for (const auto& [id, r] : ranks)
        if (id.layer > 0 && !quad_supported(8, r)) return false;
    // the two layer-1 subtrees: transfers over transfers over leaves m..m+3
    QuadArgs q[2];
    for (int side = 0; side < 2; ++side) {
        const TreeNode& root = tree.node(NodeId{1, side});
        if (root.kind != NodeKind::Transfer) return false;
        const TreeNode* mid[2];
        for (int j = 0; j < 2; ++j) {
            mid[j] = &tree.node(root.successors[static_cast<size_t>(j)]);
            if (mid[j]->kind != NodeKind::Transfer) return false;
            for (int k = 0; k < 2; ++k) {
                const TreeNode& leaf = tree.node(mid[j]->successors[static_cast<size_t>(k)]);
                if (leaf.kind != NodeKind::Leaf || leaf.leaf_dim != 4 * side + 2 * j + k) return false;
                q[side].U[2 * j + k] = h.core(leaf.id).data();
            }
        }
        q[side].T01 = h.core(mid[0]->id).data();
        q[side].T23 = h.core(mid[1]->id).data();
        q[side].T = h.core(root.id).data();
    }
    const int64_t batch = y.shape[8];
    // first half: modes 0-3 (contiguous 8^4 blocks of y) -> [8^4 (modes 4-7), 4, batch]
    if ((reinterpret_cast<uintptr_t>(y.data()) & 15u) != 0) return false;
    DT mid = c.tensor({8, 8, 8, 8, 4, batch});
    BufPtr yparts = c.alloc(c.num_sms);
    q[0].X = y.data();
    q[0].O = 4096 * batch;
    q[0].P = 4096;
    q[0].out = mid.data();
    q[0].partials = yparts->p;
    if (ev0) HTR_CUDA(cudaEventRecord(ev0, c.s));
    const int g0 = launch_quad(q[0], false, c.num_sms, c.s, &c.launches);
    if (ev1) HTR_CUDA(cudaEventRecord(ev1, c.s));
    HTR_CUDA(cudaGetLastError());
    // second half: blocks (c, s) of mid over modes 4-7 -> the latent [4, 4, batch]
    DT lat;
    if (latent_target && latent_target->shape == Shape{4, 4, batch}) {
        lat = *latent_target;
    } else {
        lat = c.tensor({4, 4, batch});
    }
    BufPtr lparts = c.alloc(c.num_sms);
    q[1].X = mid.data();
    q[1].O = 4 * batch;
    q[1].P = 4;
    q[1].out = lat.data();
    q[1].partials = lparts->p;
    q[1].ysq_partials = yparts->p;
    q[1].n_ysq = g0;
    q[1].sc = sc;
    q[1].host_out = host_out;
    q[1].ticket = c.d_ticket;
    launch_quad(q[1], true, c.num_sms, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    *latent = lat;
    return true;
}

/// Balanced 4-way trees ((1,2),(3,4)) (config 3): fused3 over the [n0, n1]
/// slabs (modes 0, 1 and ||y||^2) + the per-sample tail (k_tail4.cu).
bool launch_skip_encode4(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc, DT* latent,
                         cudaEvent_t ev0, cudaEvent_t ev1, double* host_out) {
    const DimensionTree& tree = h.tree;
    if (tree.dims() != 4 || tree.depth() != 2 || tree.layer_size(1) != 2) return false;
    const TreeNode* tr[2];
    const TreeNode* leaf[4];
    for (int side = 0; side < 2; ++side) {
        tr[side] = &tree.node(NodeId{1, side});
        if (tr[side]->kind != NodeKind::Transfer) return false;
        for (int k = 0; k < 2; ++k) {
            const TreeNode& l = tree.node(tr[side]->successors[static_cast<size_t>(k)]);
            if (l.kind != NodeKind::Leaf || l.leaf_dim != 2 * side + k) return false;
            leaf[2 * side + k] = &l;
        }
    }
    const Basis b0 = basis_of(h, leaf[0]->id), b1 = basis_of(h, leaf[1]->id), b2 = basis_of(h, leaf[2]->id),
                b3 = basis_of(h, leaf[3]->id), B12 = basis_of(h, tr[0]->id), B34 = basis_of(h, tr[1]->id);
    const int64_t n0 = y.shape[0], n1 = y.shape[1], n2 = y.shape[2], n3 = y.shape[3], batch = y.shape[4];
    const int64_t R01 = b0.r * b1.r;
    if (b0.r > 24 || b1.r > 24 || b2.r > 24 || b3.r > 24 || B12.r > 96 || B34.r > 1024 || batch < 1) return false;
    if (!fused3_supported(n0, n1, n2 * n3 * batch, static_cast<int>(b0.r), static_cast<int>(b1.r), 1) ||
        !tail4_supported(static_cast<int>(R01), static_cast<int>(B12.r), static_cast<int>(B34.r),
                         static_cast<int>(b2.r), static_cast<int>(b3.r), n2, n3) ||
        (reinterpret_cast<uintptr_t>(y.data()) & 15u) != 0)
        return false;
    DT W = c.tensor({b0.r, b1.r, n2, n3, batch});
    Fused3Args fa;
    fa.Y = y.data();
    fa.n2 = n2 * n3 * batch;
    fa.S = 1;
    fa.U0 = b0.p;
    fa.U1 = b1.p;
    fa.r0 = static_cast<int>(b0.r);
    fa.r1 = static_cast<int>(b1.r);
    fa.r2 = 1;
    fa.slab_gemm = false;
    fa.wslab = W.data();
    BufPtr parts = c.alloc(c.num_sms + static_cast<int64_t>(c.num_sms) * 24 * R01);
    fa.ysq_partials = parts->p;
    if (ev0) HTR_CUDA(cudaEventRecord(ev0, c.s));
    const int grid = launch_fused3(n0, n1, fa, c.num_sms, c.s, &c.launches);
    if (ev1) HTR_CUDA(cudaEventRecord(ev1, c.s));
    HTR_CUDA(cudaGetLastError());
    if (grid <= 0) return false;  // no tensor map for this pointer: nothing was launched
    Tail4Args ta;
    ta.W = W.data();
    ta.B12 = B12.p;
    ta.U2 = b2.p;
    ta.U3 = b3.p;
    ta.B34 = B34.p;
    ta.R01 = static_cast<int>(R01);
    ta.r12 = static_cast<int>(B12.r);
    ta.r2 = static_cast<int>(b2.r);
    ta.r3 = static_cast<int>(b3.r);
    ta.r34 = static_cast<int>(B34.r);
    ta.n2 = n2;
    ta.n3 = n3;
    ta.S = batch;
    DT lat;
    if (latent_target && latent_target->shape == Shape{B12.r, B34.r, batch}) {
        lat = *latent_target;
    } else {
        lat = c.tensor({B12.r, B34.r, batch});
    }
    ta.latent = lat.data();
    BufPtr lsq = c.alloc(batch);
    ta.latsq = lsq->p;
    ta.ysq_partials = parts->p;
    ta.n_ysq = grid;
    ta.out = sc;
    ta.host_out = host_out;
    ta.ticket = c.d_ticket;
    launch_tail4(ta, c.num_sms, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    *latent = lat;
    return true;
}

bool launch_skip_encode_fused(Context& c, const Rep& h, const DT& y, const DT* latent_target, double* sc,
                              DT* latent, cudaEvent_t ev0, cudaEvent_t ev1, double* host_out) {
    return launch_skip_encode3(c, h, y, latent_target, sc, latent, ev0, ev1, host_out) ||
           launch_skip_encode4(c, h, y, latent_target, sc, latent, ev0, ev1, host_out) ||
           launch_skip_encode8(c, h, y, latent_target, sc, latent, ev0, ev1, host_out);
}

double telescope_floor_sq(const Rep& h) {
    const double beta = 2.0 * h.defect + 16.0 * 0x1p-53;
    const double f = beta / (2.0 * kProjErrorTol);
    return f * f;
}

void measure_defect(Context& c, Rep& h) {
    std::vector<const double*> U;
    std::vector<int64_t> al, rr;
    for (Index l = 1; l <= h.tree.depth(); ++l)
        for (const TreeNode& n : h.tree.layer(l)) {
            const DT& core = h.core(n.id);
            const Basis b = basis_of(h, n.id);
            const bool ident = core.buf && core.buf->identity && core.offset == 0 && b.alpha == b.r;
            U.push_back(ident || b.r == 0 ? nullptr : b.p);
            al.push_back(b.alpha);
            rr.push_back(b.r);
        }
    if (U.empty()) {
        h.defect = 0.0;
        return;
    }
    BufPtr out = c.alloc(static_cast<int64_t>(U.size()));
    launch_basis_defect(U.data(), al.data(), rr.data(), static_cast<int>(U.size()), out->p, c.s, &c.launches);
    HTR_CUDA(cudaGetLastError());
    std::vector<double> d(U.size());
    c.fetch(out->p, static_cast<int64_t>(d.size()), d.data());
    double sum = 0.0;
    for (double v : d) sum += v;
    h.defect = sum;
}

double residual_sq_global(Context& c, const Rep& h, const DT& latent, const DT& y) {
    BufPtr r = c.alloc(1);
    decode_residual_sq(c, h, latent, y, r->p);
    c.allreduce(r->p, 1);
    double v = 0.0;
    c.fetch(r->p, 1, &v);
    return v;
}

EncodeOut encode(Context& c, const Rep& h, const DT& y, bool exact, const DT* latent_target, double* sc_deferred) {
    const DimensionTree& tree = h.tree;
    const Index d = tree.dims(), p = tree.depth();
    const int64_t batch = y.shape[static_cast<size_t>(d)];
    EncodeOut out;
    out.exact = exact;
    const RankMap ranks = h.ranks();
    // [0] ysq, [1] nonfinite, [2] latent^2, [16..] step energies
    double* sc = sc_deferred ? sc_deferred : c.d_sc->p;
    int nslots = 0;
    // (the context's events and mapped block are not per call: a deferred
    // encode uses neither)
    const bool prof = c.profile && !sc_deferred;
    double* host_out = (c.sharded() || sc_deferred) ? nullptr : c.d_map;
    // the generic kernels accumulate into the scalar slots; the fused
    // leaf+tail path assigns sc[0] and sc[2] and needs no clearing
    bool zeroed = false;
    auto zero_scalars = [&] {
        if (!zeroed) HTR_CUDA(cudaMemsetAsync(sc, 0, (sc_deferred ? 16 : 512) * sizeof(double), c.s));
        zeroed = true;
    };

    // sharded: every rank all-reduces the same 16 + nslots slots, whichever
    // kernels its shard took, so none may hold stale values (the fused
    // kernels assign only sc[0] and sc[2])
    if (c.sharded()) zero_scalars();
    DT cur = y;
    bool leaves_done = false;
    bool tail_done = false;  // latent and ||latent||^2 already produced
    if (!exact && c.fused && d == 3) {
        DT lat;
        if (launch_skip_encode3(c, h, y, latent_target, sc, &lat, prof ? c.ev[0] : nullptr,
                                prof ? c.ev[1] : nullptr, host_out)) {
            // fused leaves + tail: ((1,(2,3)) trees)
            leaves_done = tail_done = out.fused = true;
            cur = lat;
        } else {
            const Tree3 t = tree3_ranks(h, ranks);
            zero_scalars();
            if (fused3_supported(y.shape[0], y.shape[1], y.shape[2], t.r0, t.r1, t.r2)) {
                // fused leaves, slab-axis GEMM, then the generic interior projections
                Fused3Args fa;
                fa.Y = y.data();
                fa.n2 = y.shape[2];
                fa.S = batch;
                fa.U0 = h.core(t.leaf_of[0]).data();
                fa.U1 = h.core(t.leaf_of[1]).data();
                fa.U2 = h.core(t.leaf_of[2]).data();
                fa.r0 = t.r0;
                fa.r1 = t.r1;
                fa.r2 = t.r2;
                DT Z = c.tensor({t.r0, t.r1, t.r2, batch});
                fa.Z = Z.data();
                fa.slab_gemm = true;
                const int64_t ws =
                    fused3_workspace_doubles(y.shape[0], y.shape[1], fa.n2, batch, t.r0, t.r1, t.r2, c.num_sms);
                BufPtr w = c.alloc(ws);
                fa.wslab = w->p;
                fa.ysq_partials = w->p + fa.n2 * batch * static_cast<int64_t>(t.r0) * t.r1;
                if (prof) HTR_CUDA(cudaEventRecord(c.ev[0], c.s));
                const int grid = launch_fused3(y.shape[0], y.shape[1], fa, c.num_sms, c.s, &c.launches);
                if (prof) HTR_CUDA(cudaEventRecord(c.ev[1], c.s));
                HTR_CUDA(cudaGetLastError());
                if (grid > 0) {  // else (no tensor map for this pointer): generic kernels below
                    launch_sum_partials(fa.ysq_partials, grid, sc + 0, c.s, &c.launches);
                    leaves_done = true;
                    out.fused = true;
                    cur = Z;
                }
            }
        }
    } else if (!exact && c.fused && (d == 8 || d == 4)) {
        DT lat;
        if (d == 8 ? launch_skip_encode8(c, h, y, latent_target, sc, &lat, prof ? c.ev[0] : nullptr,
                                         prof ? c.ev[1] : nullptr, host_out)
                   : launch_skip_encode4(c, h, y, latent_target, sc, &lat, prof ? c.ev[0] : nullptr,
                                         prof ? c.ev[1] : nullptr, host_out)) {
            leaves_done = tail_done = out.fused = true;
            cur = lat;
        }
    }
    bool ysq_fused = false;  // ||y||^2 taken during the first projection (one read of y)
    if (!leaves_done) {
        zero_scalars();
        const std::vector<TreeNode>& lay = tree.layer(p);
        for (size_t q = 0; q < lay.size();) {
            const TreeNode& n = lay[q];
            const int mode = static_cast<int>(n.leaf_dim);
            const bool first = q == 0;
            if (!exact && c.fused && first && mode == 0 && q + 1 < lay.size() && lay[q + 1].kind == NodeKind::Leaf &&
                lay[q + 1].leaf_dim == 1) {
                // leaves of modes 0 and 1 in one pass on the FP64 tensor cores:
                // fused3 over [n0, n1, rest] slabs writes the projected tensor
                // (r0 x r1 per slab, canonical) and ||y||^2 (config 3)
                const Basis b0 = basis_of(h, n.id), b1 = basis_of(h, lay[q + 1].id);
                const int64_t J0 = cur.shape[0], J1 = cur.shape[1];
                const int64_t rest = cur.size() / (J0 * J1);
                if (fused3_supported(J0, J1, rest, static_cast<int>(b0.r), static_cast<int>(b1.r), 1) &&
                    (reinterpret_cast<uintptr_t>(cur.data()) & 15u) == 0) {
                    Shape os = cur.shape;
                    os[0] = b0.r;
                    os[1] = b1.r;
                    DT lo = c.tensor(os);
                    Fused3Args fa;
                    fa.Y = cur.data();
                    fa.n2 = rest;
                    fa.S = 1;
                    fa.U0 = b0.p;
                    fa.U1 = b1.p;
                    fa.r0 = static_cast<int>(b0.r);
                    fa.r1 = static_cast<int>(b1.r);
                    fa.r2 = 1;
                    fa.slab_gemm = false;
                    fa.wslab = lo.data();
                    const int64_t R01 = b0.r * b1.r;
                    BufPtr parts = c.alloc(c.num_sms + static_cast<int64_t>(c.num_sms) * 24 * R01);
                    fa.ysq_partials = parts->p;
                    if (prof) HTR_CUDA(cudaEventRecord(c.ev[0], c.s));
                    const int grid = launch_fused3(J0, J1, fa, c.num_sms, c.s, &c.launches);
                    if (prof) HTR_CUDA(cudaEventRecord(c.ev[1], c.s));
                    HTR_CUDA(cudaGetLastError());
                    if (grid > 0) {
                        launch_sum_partials(parts->p, grid, sc + 0, c.s, &c.launches);
                        ysq_fused = true;
                        out.fused = true;
                        cur = lo;
                        q += 2;
                        continue;
                    }
                }
            }
            if (!exact && c.fused && q + 1 < lay.size() && lay[q + 1].kind == NodeKind::Leaf &&
                lay[q + 1].leaf_dim == n.leaf_dim + 1) {
                // two adjacent small leaves in one pass over the tensor
                const Basis b0 = basis_of(h, n.id), b1 = basis_of(h, lay[q + 1].id);
                int64_t I = 1, O = 1;
                for (int k = 0; k < mode; ++k) I *= cur.shape[static_cast<size_t>(k)];
                for (size_t k = static_cast<size_t>(mode) + 2; k < cur.shape.size(); ++k) O *= cur.shape[k];
                const int64_t J0 = cur.shape[static_cast<size_t>(mode)], J1 = cur.shape[static_cast<size_t>(mode) + 1];
                if (J0 <= 8 && J1 <= 8 && b0.r <= 4 && b1.r <= 4 && I * O >= 4096) {
                    Shape os = cur.shape;
                    os[static_cast<size_t>(mode)] = b0.r;
                    os[static_cast<size_t>(mode) + 1] = b1.r;
                    DT out = c.tensor(os);
                    BufPtr yp = first ? c.alloc(8 * c.num_sms) : nullptr;
                    const int nb = launch_pair_project(cur.data(), I, J0, J1, O, b0.p, b0.r, b1.p, b1.r, out.data(),
                                                       yp ? yp->p : nullptr, c.num_sms, c.s, &c.launches);
                    if (nb > 0) {
                        HTR_CUDA(cudaGetLastError());
                        if (yp) {
                            launch_sum_partials(yp->p, nb, sc + 0, c.s, &c.launches);
                            ysq_fused = true;
                        }
                        cur = out;
                        q += 2;
                        continue;
                    }
                }
            }
            bool done = false;
            cur = project(c, cur, mode, basis_of(h, n.id), exact ? sc + 16 + nslots++ : nullptr,
                          first ? sc + 0 : nullptr, first ? &done : nullptr);
            if (first) ysq_fused = done;
            ++q;
        }
    }
    for (Index l = p - 1; l >= 1 && !tail_done; --l) {
        cur.shape = layer_extents(h, l, ranks, batch, leaves_done);
        // the last projection of layer 1 yields the latent: written into the
        // root store's next slices when the caller provides them
        Index last = -1;
        for (Index j = 0; j < tree.layer_size(l); ++j)
            if (!(leaves_done && tree.layer(l)[static_cast<size_t>(j)].kind == NodeKind::Leaf)) last = j;
        for (Index j = 0; j < tree.layer_size(l); ++j) {
            const TreeNode& n = tree.layer(l)[static_cast<size_t>(j)];
            if (leaves_done && n.kind == NodeKind::Leaf) continue;
            const DT* dst = (l == 1 && j == last && !exact) ? latent_target : nullptr;
            cur = project(c, cur, static_cast<int>(j), basis_of(h, n.id), exact ? sc + 16 + nslots++ : nullptr,
                          nullptr, nullptr, dst);
        }
    }
    out.latent = cur;

    // ||y||^2 unless the fused kernel produced it, plus ||latent||^2
    BufPtr parts = c.alloc(kReduceBlocks);
    const bool ysq_scanned = !leaves_done && !ysq_fused;  // sumsq also flags non-finite input
    if (ysq_scanned) {
        launch_sumsq(y.data(), y.size(), parts->p, sc + 0, c.s, &c.launches);
    }
    BufPtr parts2 = c.alloc(kReduceBlocks);
    if (!tail_done) launch_sumsq(cur.data(), cur.size(), parts2->p, sc + 2, c.s, &c.launches);  // sc[2], sc[3]
    HTR_CUDA(cudaGetLastError());
    if (sc_deferred) {
        out.scan_valid = ysq_scanned;
        return out;
    }
    if (c.sharded()) {
        // the global batch count rides on the same all-reduce (slot 8)
        c.h_sc[8] = static_cast<double>(batch);
        HTR_CUDA(cudaMemcpyAsync(sc + 8, c.h_sc + 8, sizeof(double), cudaMemcpyHostToDevice, c.s));
    }
    if (tail_done && !c.sharded()) {
        // the fused tail wrote both norms to mapped host memory
        HTR_CUDA(cudaStreamSynchronize(c.s));
        c.h_sc[0] = c.h_map[0];
        c.h_sc[1] = 0.0;  // no full scan ran
        c.h_sc[2] = c.h_map[2];
    } else {
        c.allreduce(sc, 16 + nslots);
        c.fetch(sc, 16 + nslots, c.h_sc);
    }
    out.gbatch = c.sharded() ? static_cast<int64_t>(std::llround(c.h_sc[8])) : batch;
    if (prof && leaves_done) {
        float ms = 0.f;
        HTR_CUDA(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
        c.fused_ms += ms;
        ++c.fused_calls;
    }
    out.ysq = c.h_sc[0];
    // sc[1]: (all-reduced) count of full scans that met a non-finite element;
    // zero where no scan ran. Both it and ||y||^2 are global, so the rescan
    // below (a collective) runs on every rank or on none.
    out.nonfinite = c.h_sc[1] != 0.0;
    const double latsq = c.h_sc[2];
    if (exact) {
        double loss = 0.0;
        for (int i = 0; i < nslots; ++i) loss += c.h_sc[16 + i];
        out.proj_sq = loss;
    } else {
        out.proj_sq = std::max(0.0, out.ysq - latsq);
    }
    if (!exact && !out.nonfinite && std::isfinite(out.ysq) && out.proj_sq < telescope_floor_sq(h) * out.ysq) {
        // below the floor the telescoped loss's square root could drift from
        // the reference's explicit-residual value (bht.hpp:357-365) by more
        // than kProjErrorTol ||y||, so the loss is re-measured as
        // ||y - decode(latent)||^2 (the same quantity: the step residuals of
        // nested orthogonal projections add up to it), one more read of y
        out.proj_sq = residual_sq_global(c, h, out.latent, y);
        out.exact = true;
    }
    if (!out.nonfinite && !std::isfinite(out.ysq)) {
        // inf/nan in ||y||^2 without a scan's flag: distinguish overflow from
        // non-finite input with the explicit scan
        double s = 0.0;
        bool bad = false;
        norm_sq(c, y.data(), y.size(), &s, &bad);
        out.nonfinite = bad;
        out.ysq = s;
    }
    return out;
}

// ---------------------------------------------------------------------------
// root append / pad
// ---------------------------------------------------------------------------

void append_root(Context& c, Rep& out, const Rep& in, const DT& latent) {
    const int64_t r11 = latent.shape[0], r12 = latent.shape[1], n = latent.shape[2];
    const std::shared_ptr<RootStore>& rs = in.root;
    const int64_t slice = r11 * r12;
    if (rs && rs->r11 == r11 && rs->r12 == r12 && rs->committed == in.acc && in.acc + n <= rs->cap) {
        // tip of the shared store: append in place, O(batch); nothing to
        // copy when the encoder already wrote the latent into the slot
        if (latent.buf != rs->buf || latent.offset != slice * in.acc)
            HTR_CUDA(cudaMemcpyAsync(rs->buf->p + slice * in.acc, latent.data(), sizeof(double) * static_cast<size_t>(slice * n),
                                 cudaMemcpyDeviceToDevice, c.s));
        rs->committed = in.acc + n;
        out.root = rs;
    } else {
        const int64_t cap = std::max<int64_t>(2 * (in.acc + n), rs ? rs->cap : 0);
        auto ns = new_root(c, r11, r12, cap);
        if (in.acc > 0) {
            if (!rs || rs->r11 != r11 || rs->r12 != r12) raise(HTR_ERR_RUNTIME, "append_root: rank mismatch");
            HTR_CUDA(cudaMemcpyAsync(ns->buf->p, rs->buf->p, sizeof(double) * static_cast<size_t>(slice * in.acc),
                                     cudaMemcpyDeviceToDevice, c.s));
        }
        HTR_CUDA(cudaMemcpyAsync(ns->buf->p + slice * in.acc, latent.data(), sizeof(double) * static_cast<size_t>(slice * n),
                                 cudaMemcpyDeviceToDevice, c.s));
        ns->committed = in.acc + n;
        out.root = ns;
    }
    out.acc = in.acc + n;
}

// ---------------------------------------------------------------------------
// HT-RISE update (ht_rise.hpp:99-186)
// ---------------------------------------------------------------------------


UpdateOut ht_rise_update(Context& c, const Rep& h, const DT& y, double eps_override, bool adaptive) {
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t l0 = c.launches;
    check_batch_input(y.shape, h.tree, &h.dims, "ht_rise_update");
    const DimensionTree& tree = h.tree;
    const Index d = tree.dims(), p = tree.depth();
    const int64_t batch = y.shape[static_cast<size_t>(d)];
    const double eps_rel = effective_eps_rel(eps_override >= 0 ? eps_override : h.eps_rel);

    UpdateOut res;
    std::memset(&res.report, 0, sizeof(res.report));
    htr_update_report& rep = res.report;

    // the latent of a skipped batch lands in the root store's next slices:
    // written there speculatively when this value is the store's tip
    DT slot;
    const DT* target = nullptr;
    if (const auto& rs = h.root; rs && rs->committed == h.acc && h.acc + batch <= rs->cap) {
        slot.buf = rs->buf;
        slot.shape = {rs->r11, rs->r12, batch};
        slot.offset = rs->r11 * rs->r12 * h.acc;
        target = &slot;
    }
    EncodeOut enc = encode(c, h, y, c.exact_loss, target);
    if (enc.nonfinite) raise(HTR_ERR_INVALID_ARGUMENT, "ht_rise_update: non-finite input");
    double norm_y = std::sqrt(enc.ysq);
    rep.eps_des = eps_rel * norm_y;
    if (!enc.exact) {
        // guard band around the skip threshold: the telescoped loss
        // ||y||^2 - ||latent||^2 carries ~u*||y||^2 absolute error, so a
        // decision that close to the boundary is re-taken with the
        // reference's explicit per-step residuals (bht.hpp:357-365)
        const double guard = 1e-12 * enc.ysq;
        if (std::abs(enc.proj_sq - rep.eps_des * rep.eps_des) <= guard) {
            enc = encode(c, h, y, true);
        }
    }
    rep.proj_error = std::sqrt(enc.proj_sq);
    rep.used_fused_path = enc.fused ? 1 : 0;
    rep.used_exact_loss = enc.exact ? 1 : 0;
    const int64_t gbatch = enc.gbatch;

    auto finish = [&](std::shared_ptr<Rep> out) {
        RankMap nr = out->ranks();
        RankMap old = h.ranks();
        int i = 0;
        for (const auto& [id, r] : nr) {
            if (i >= HTR_MAX_NODES) break;
            rep.node_layer[i] = static_cast<int32_t>(id.layer);
            rep.node_pos[i] = static_cast<int32_t>(id.pos);
            rep.new_ranks[i] = r;
            rep.added_ranks[i] = r - old.at(id);
            ++i;
        }
        rep.n_nodes = i;
        out->acc_global = h.acc_global + gbatch;
        HTR_CUDA(cudaStreamSynchronize(c.s));
        rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        rep.kernel_launches = c.launches - l0;
        res.rep = std::move(out);
        return res;
    };

    if (rep.proj_error <= rep.eps_des) {
        rep.skipped = 1;
        auto out = std::make_shared<Rep>(h);
        append_root(c, *out, h, enc.latent);
        return finish(out);
    }

    // ---- EXPAND ----------------------------------------------------------
    auto out = std::make_shared<Rep>(h);
    RankMap ranks = h.ranks();
    double eps_nw = rep.eps_des / std::sqrt(static_cast<double>(2 * d - 2));
    const double ysq = enc.ysq;
    const double col_scale = static_cast<double>(gbatch) / static_cast<double>(batch);
    // the root is re-padded lazily: remember pending layer-1 growth
    int64_t pad0 = 0, pad1 = 0;

    auto expand_node = [&](const TreeNode& n, const Basis& U, const Truncation& tb) {
        if (tb.rank == 0) return;
        // re-orthonormalise the new directions against the old basis and
        // append (expand_core, ht_rise.hpp:53-79)
        BufPtr info = c.alloc(4);
        BufPtr work = c.alloc(U.r * tb.rank + tb.rank * tb.rank + 16);
        launch_orthonormalize_new(U.p, U.alpha, U.r, tb.u.data(), tb.rank, info->p, work->p, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        double hinfo[2];
        c.fetch(info->p, 2, hinfo);
        if (!(hinfo[0] <= 1e-8 * std::max(1.0, hinfo[1])))
            raise(HTR_ERR_INVALID_ARGUMENT, "expand_core: new directions not orthogonal to existing basis (defect " +
                                                std::to_string(hinfo[0]) + ")");
        const int64_t rn = U.r + tb.rank;
        DT joined = c.tensor({U.alpha, rn});
        HTR_CUDA(cudaMemcpyAsync(joined.data(), U.p, sizeof(double) * static_cast<size_t>(U.alpha * U.r),
                                 cudaMemcpyDeviceToDevice, c.s));
        HTR_CUDA(cudaMemcpyAsync(joined.data() + U.alpha * U.r, tb.u.data(),
                                 sizeof(double) * static_cast<size_t>(U.alpha * tb.rank), cudaMemcpyDeviceToDevice, c.s));
        if (n.kind != NodeKind::Leaf) {
            const Shape& s = out->core(n.id).shape;
            joined.shape = {s[0], s[1], rn};
        }
        out->cores[static_cast<size_t>(n.id.layer)][static_cast<size_t>(n.id.pos)] = joined;
        ranks[n.id] += tb.rank;
        // pad the parent's successor slot with zeros (pad_with_zeros, ht_rise.hpp:83-92)
        const Index slot = tree.parent_slot(n.id);
        const TreeNode& par = tree.node(n.parent);
        if (par.kind == NodeKind::Root) {
            (slot == 0 ? pad0 : pad1) += tb.rank;
        } else {
            const DT& pc = out->core(n.parent);
            const int64_t inner = slot == 0 ? 1 : pc.shape[0];
            const int64_t ext = pc.shape[static_cast<size_t>(slot)];
            const int64_t outer = slot == 0 ? pc.shape[1] * pc.shape[2] : pc.shape[2];
            Shape ns = pc.shape;
            ns[static_cast<size_t>(slot)] += tb.rank;
            DT padded = c.tensor(ns);
            launch_pad_axis(pc.data(), inner, ext, outer, tb.rank, padded.data(), c.s, &c.launches);
            HTR_CUDA(cudaGetLastError());
            out->cores[static_cast<size_t>(n.parent.layer)][static_cast<size_t>(n.parent.pos)] = padded;
        }
    };

    // every node of a layer truncates its residual against the same working
    // tensor (ht_rise.hpp:157-162: all nodes expand, then all project), so the
    // layer's truncations run first (eigensolves batched), then the expansions
    auto expand_layer = [&](const std::vector<TreeNode>& nodes, const DT& cur, bool leaves) {
        std::vector<int> modes;
        std::vector<int64_t> cols;
        std::vector<Basis> olds;
        for (size_t j = 0; j < nodes.size(); ++j) {
            const int mode = leaves ? static_cast<int>(nodes[j].leaf_dim) : static_cast<int>(j);
            modes.push_back(mode);
            cols.push_back(static_cast<int64_t>(
                std::llround(static_cast<double>(cur.size() / cur.shape[static_cast<size_t>(mode)]) * col_scale)));
            olds.push_back(basis_of(*out, nodes[j].id));
        }
        std::vector<Truncation> tbs = truncate_modes(c, cur, modes, eps_nw, 0, cols, true, false, &olds);
        for (size_t j = 0; j < nodes.size(); ++j) expand_node(nodes[j], olds[j], tbs[j]);
    };

    DT cur = y;
    expand_layer(tree.layer(p), cur, true);
    {
        std::vector<Basis> lb;
        for (const TreeNode& n : tree.layer(p)) lb.push_back(basis_of(*out, n.id));
        cur = project_leaves(c, cur, tree.layer(p), lb);
    }

    for (Index l = p - 1; l >= 1; --l) {
        if (adaptive) {
            double cn2 = 0.0;
            norm_sq(c, cur.data(), cur.size(), &cn2, nullptr);
            eps_nw = adaptive_budget(rep.eps_des, std::max(0.0, ysq - cn2), svds_below(tree, l + 1));
        }
        cur.shape = layer_extents(*out, l, ranks, batch, false);
        expand_layer(tree.layer(l), cur, false);
        for (Index j = 0; j < tree.layer_size(l); ++j)
            cur = project(c, cur, static_cast<int>(j), basis_of(*out, tree.layer(l)[static_cast<size_t>(j)].id), nullptr);
    }

    // root: zero-pad the stored slices to the grown layer-1 ranks, then append
    if (pad0 || pad1) {
        const std::shared_ptr<RootStore>& rs = h.root;
        const int64_t r11 = rs->r11 + pad0, r12 = rs->r12 + pad1;
        auto ns = new_root(c, r11, r12, std::max<int64_t>(rs->cap, 2 * (h.acc + batch)));
        if (h.acc > 0) {
            BufPtr tmp = c.alloc(r11 * rs->r12 * h.acc);
            // axis 0 then axis 1 of [r11_old, r12_old, acc]
            launch_pad_axis(rs->buf->p, 1, rs->r11, rs->r12 * h.acc, pad0, tmp->p, c.s, &c.launches);
            launch_pad_axis(tmp->p, r11, rs->r12, h.acc, pad1, ns->buf->p, c.s, &c.launches);
            HTR_CUDA(cudaGetLastError());
        }
        ns->committed = h.acc;
        Rep padded_in = h;
        padded_in.root = ns;
        out->root = ns;
        append_root(c, *out, padded_in, cur);
    } else {
        append_root(c, *out, h, cur);
    }
    measure_defect(c, *out);
    return finish(out);
}

// ---------------------------------------------------------------------------
// stream of updates (extension; the reference's CLI loops ht_rise_update over
// batches, main.cpp:225-243): skip-path encodes pipelined one batch ahead
// ---------------------------------------------------------------------------

std::vector<UpdateOut> ht_rise_update_many(Context& c, const std::shared_ptr<Rep>& h0, int64_t n,
                                           const std::function<DT(int64_t)>& batch_of, double eps_override,
                                           bool adaptive) {
    const auto t_entry = std::chrono::steady_clock::now();
    std::vector<UpdateOut> res;
    res.reserve(static_cast<size_t>(std::max<int64_t>(n, 0)));
    std::shared_ptr<Rep> cur = h0;
    const Index d = h0->tree.dims();
    // one launched-but-undecided skip-path encode
    struct Slot {
        int64_t index = -1;
        DT y, latent;
        BufPtr dsc;       // [0] ||y||^2, [1] non-finite flag, [2] ||latent||^2, [8] batch count (sharded)
        double* host = nullptr;  // pinned copy of dsc[0..8]
        double* mapped = nullptr;  // mapped host block the tail writes dsc[0], dsc[2] to
        bool fused = false;        // launched through the fused skip-path kernels
        bool used_fused = false;   // (report) any fused kernel in the encode
        bool scan_valid = false;   // dsc[1] is the non-finite flag of a full scan
        bool resid = false;        // dsc[4] holds ||y - decode(latent)||^2 (explicit loss, enqueued ahead)
        bool resid_mapped = false;  // ... and the kernel mirrored it into mapped[4]
        bool from_mapped = false;   // the decision reads the mapped block (no device-to-host copy)
        cudaEvent_t done = nullptr, t0 = nullptr, t1 = nullptr;
        int64_t launches = 0;
        std::chrono::steady_clock::time_point started;
    };
    Slot slots[2];
    bool refine_hint = false;  // the last decided batch needed the explicit loss
    // HTR_TIMELINE=1: device timeline of the stream (events around each
    // launch), printed to stderr at the end (diagnostics only)
    static const bool timeline = std::getenv("HTR_TIMELINE") != nullptr;
    std::vector<cudaEvent_t> tl;
    auto mark = [&] {
        if (!timeline) return;
        cudaEvent_t e;
        HTR_CUDA(cudaEventCreate(&e));
        HTR_CUDA(cudaEventRecord(e, c.s));
        tl.push_back(e);
    };
    for (int k = 0; k < 2; ++k) {
        slots[k].host = c.h_sc + 960 + 16 * k;
        slots[k].mapped = c.h_map + 16 + 16 * k;
        slots[k].done = c.slot_ev[k][0];
        slots[k].t0 = c.slot_ev[k][1];
        slots[k].t1 = c.slot_ev[k][2];
    }

    // batches are fetched once each, in order; at most two are held
    DT held[2];
    int64_t held_idx[2] = {-1, -1};
    auto batch = [&](int64_t i) -> DT {
        for (int k = 0; k < 2; ++k)
            if (held_idx[k] == i) return held[k];
        const int k = held_idx[0] < held_idx[1] ? 0 : 1;  // evict the older
        held[k] = batch_of(i);
        held_idx[k] = i;
        check_batch_input(held[k].shape, cur->tree, &cur->dims, "ht_rise_update");
        return held[k];
    };

    // launch batch i against h's bases with its latent at root slice `at`
    auto launch = [&](Slot& sl, const Rep& h, int64_t i, int64_t at) -> bool {
        sl.index = -1;
        if (c.exact_loss) return false;  // per-step energies: the per-call path
        sl.y = batch(i);
        const int64_t nb = sl.y.shape[static_cast<size_t>(d)];
        DT slot;
        const DT* target = nullptr;
        if (const auto& rs = h.root; rs && rs->committed == h.acc && at + nb <= rs->cap) {
            slot.buf = rs->buf;
            slot.shape = {rs->r11, rs->r12, nb};
            slot.offset = rs->r11 * rs->r12 * at;
            target = &slot;
        }
        const int64_t l0 = c.launches;
        sl.started = std::chrono::steady_clock::now();
        sl.dsc = c.alloc(16);  // [0] ||y||^2, [1] non-finite flag, [2] ||latent||^2, [8] batch count
        // sharded: all ranks reduce the block whichever path their shard
        // took, so it starts zeroed (the fused kernels assign [0] and [2] only)
        if (c.sharded()) HTR_CUDA(cudaMemsetAsync(sl.dsc->p, 0, 16 * sizeof(double), c.s));
        mark();
        double* mapped_dev = c.d_map + (sl.mapped - c.h_map);
        sl.fused = c.fused && launch_skip_encode_fused(c, h, sl.y, target, sl.dsc->p, &sl.latent,
                                                       c.profile ? sl.t0 : nullptr, c.profile ? sl.t1 : nullptr,
                                                       c.sharded() ? nullptr : mapped_dev);
        sl.used_fused = sl.fused;
        sl.scan_valid = false;
        if (!sl.fused) {
            // any other tree: the per-call encode, enqueued only (its scalars
            // land in the slot's block and are read back below)
            EncodeOut e = encode(c, h, sl.y, false, target, sl.dsc->p);
            sl.latent = e.latent;
            sl.used_fused = e.fused;
            sl.scan_valid = e.scan_valid;
        }
        // the explicit loss, enqueued behind the encode when the previous
        // batch needed it (its telescoped loss sat below the accuracy floor,
        // as every batch of a stream near the floor does): the decision then
        // reads it without another host round trip
        sl.resid = refine_hint;
        // (the fused reconstruction kernel mirrors it into the slot's mapped block)
        sl.resid_mapped = false;
        if (sl.resid)
            sl.resid_mapped = decode_residual_sq(c, h, sl.latent, sl.y, sl.dsc->p + 4,
                                                 c.sharded() ? nullptr : mapped_dev + 4);
        if (c.sharded()) {
            // the global batch count rides on the skip test's all-reduce
            sl.host[8] = static_cast<double>(nb);
            HTR_CUDA(cudaMemcpyAsync(sl.dsc->p + 8, sl.host + 8, sizeof(double), cudaMemcpyHostToDevice, c.s));
            c.allreduce(sl.dsc->p, 9);
        }
        sl.from_mapped = !c.sharded() && sl.fused && (!sl.resid || sl.resid_mapped);
        if (!sl.from_mapped)
            HTR_CUDA(cudaMemcpyAsync(sl.host, sl.dsc->p, 9 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
        HTR_CUDA(cudaEventRecord(sl.done, c.s));
        mark();
        sl.launches = c.launches - l0;
        sl.index = i;
        return true;
    };

    // the skip decision of a launched batch (ht_rise_update's, bit for bit);
    // null when the batch needs the full update (expansion, guard band,
    // non-finite input)
    auto decide = [&](Slot& sl, const Rep& h) -> std::shared_ptr<Rep> {
        HTR_CUDA(cudaEventSynchronize(sl.done));
        const int64_t nb = sl.y.shape[static_cast<size_t>(d)];
        const double* v = sl.from_mapped ? sl.mapped : sl.host;
        const double ysq = v[0], latsq = v[2];
        const int64_t gbatch = c.sharded() ? static_cast<int64_t>(std::llround(v[8])) : nb;
        // non-finite input (the per-call path raises); sharded, the flag is
        // the all-reduced count, identical on every rank
        if ((c.sharded() || sl.scan_valid) && v[1] != 0.0) return nullptr;
        if (c.profile && sl.fused) {
            float ms = 0.f;
            HTR_CUDA(cudaEventElapsedTime(&ms, sl.t0, sl.t1));
            c.fused_ms += ms;
            ++c.fused_calls;
        }
        if (!std::isfinite(ysq)) return nullptr;
        const double eps_rel = effective_eps_rel(eps_override >= 0 ? eps_override : h.eps_rel);
        const double eps_des = eps_rel * std::sqrt(ysq);
        double proj_sq = std::max(0.0, ysq - latsq);
        bool refined = false;
        if (proj_sq < telescope_floor_sq(h) * ysq) {  // as in encode(): re-measure explicitly
            proj_sq = sl.resid ? v[4] : residual_sq_global(c, h, sl.latent, sl.y);
            refined = true;
        }
        refine_hint = refined;
        if (std::abs(proj_sq - eps_des * eps_des) <= 1e-12 * ysq) return nullptr;
        const double proj_error = std::sqrt(proj_sq);
        if (!(proj_error <= eps_des)) return nullptr;
        auto out = std::make_shared<Rep>(h);
        append_root(c, *out, h, sl.latent);
        out->acc_global = h.acc_global + gbatch;
        UpdateOut u;
        std::memset(&u.report, 0, sizeof(u.report));
        htr_update_report& r = u.report;
        r.skipped = 1;
        r.proj_error = proj_error;
        r.eps_des = eps_des;
        r.used_fused_path = sl.used_fused ? 1 : 0;
        r.used_exact_loss = refined ? 1 : 0;
        int k = 0;
        for (const auto& [id, rk] : out->ranks()) {
            if (k >= HTR_MAX_NODES) break;
            r.node_layer[k] = static_cast<int32_t>(id.layer);
            r.node_pos[k] = static_cast<int32_t>(id.pos);
            r.new_ranks[k] = rk;
            r.added_ranks[k] = 0;
            ++k;
        }
        r.n_nodes = k;
        r.kernel_launches = sl.launches;
        r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - sl.started).count();
        u.rep = out;
        res.push_back(std::move(u));
        return out;
    };

    int cs = 0;          // slot of batch i when `pending`
    bool pending = false;
    std::chrono::steady_clock::time_point t_first = t_entry;
    for (int64_t i = 0; i < n; ++i) {
        if (!pending) pending = launch(slots[cs], *cur, i, cur->acc);
        if (i == 0) t_first = std::chrono::steady_clock::now();
        if (!pending) {
            UpdateOut u = ht_rise_update(c, *cur, batch(i), eps_override, adaptive);
            cur = u.rep;
            res.push_back(std::move(u));
            continue;
        }
        // batch i+1 against the same bases, its latent right after batch i's
        const bool ahead =
            i + 1 < n && launch(slots[cs ^ 1], *cur, i + 1, cur->acc + slots[cs].y.shape[static_cast<size_t>(d)]);
        if (auto next = decide(slots[cs], *cur)) {
            cur = next;
            cs ^= 1;
            pending = ahead;
        } else {
            // expansion (or a decision inside the guard band): the full
            // update; a speculative batch i+1 is discarded (its latent went to
            // slices beyond the committed ones) and re-runs on the new bases
            UpdateOut u = ht_rise_update(c, *cur, slots[cs].y, eps_override, adaptive);
            cur = u.rep;
            res.push_back(std::move(u));
            pending = false;
        }
        slots[cs ^ 1].dsc.reset();
    }
    HTR_CUDA(cudaStreamSynchronize(c.s));
    if (timeline) {
        const auto us = [&](std::chrono::steady_clock::time_point t) {
            return std::chrono::duration<double, std::micro>(t - t_entry).count();
        };
        std::fprintf(stderr, "timeline host: first launch done %.1f us, exit %.1f us\n",
                     res.empty() ? 0.0 : us(t_first), us(std::chrono::steady_clock::now()));
    }
    if (timeline && tl.size() >= 2) {
        for (size_t k = 0; k + 1 < tl.size(); k += 2) {
            float busy = 0.f, gap = 0.f;
            HTR_CUDA(cudaEventElapsedTime(&busy, tl[k], tl[k + 1]));
            if (k + 2 < tl.size()) HTR_CUDA(cudaEventElapsedTime(&gap, tl[k + 1], tl[k + 2]));
            std::fprintf(stderr, "timeline launch %zu: %.4f ms, then %.4f ms to the next\n", k / 2, busy, gap);
        }
        for (cudaEvent_t e : tl) cudaEventDestroy(e);
    }
    return res;
}


// ---------------------------------------------------------------------------
// decode (bht.hpp:406-456)
// ---------------------------------------------------------------------------

namespace {
DT decode_impl(Context& c, const Rep& h, const DT& latent, double* dst, const DT* ref, double* resid_out,
               double* resid_host = nullptr, bool* host_written = nullptr);
}

DT decode(Context& c, const Rep& h, const DT& latent, double* dst) { return decode_impl(c, h, latent, dst, nullptr, nullptr); }

bool decode_residual_sq(Context& c, const Rep& h, const DT& latent, const DT& y, double* out, double* host_out) {
    bool written = false;
    decode_impl(c, h, latent, nullptr, &y, out, host_out, &written);
    return written;
}

namespace {
DT decode_impl(Context& c, const Rep& h, const DT& latent, double* dst, const DT* ref, double* resid_out,
               double* resid_host, bool* host_written) {
    const int64_t r11 = h.root->r11, r12 = h.root->r12;
    if (latent.shape.size() != 3 || latent.shape[0] != r11 || latent.shape[1] != r12)
        raise(HTR_ERR_INVALID_ARGUMENT, "decode: latent ranks " + htrise::shape_to_string(latent.shape) +
                                            " do not match root [" + std::to_string(r11) + "x" + std::to_string(r12) + "]");
    // The mode products of bht.hpp:406-456 act on distinct modes and commute.
    // Transfer nodes (which do not grow the tensor) are expanded top-down
    // first; the leaf factors, each growing its mode from r to n, follow in
    // order of increasing growth, so every product runs on the smallest
    // tensor it can. The last product writes into dst.
    std::vector<NodeId> modes = {h.tree.node({0, 0}).successors[0], h.tree.node({0, 0}).successors[1]};
    DT cur = latent;
    for (bool split = true; split;) {
        split = false;
        for (size_t pos = 0; pos < modes.size(); ++pos) {
            const TreeNode& n = h.tree.node(modes[pos]);
            if (n.kind != NodeKind::Transfer) continue;
            const Basis b = basis_of(h, n.id);
            // multiply mode `pos` by the basis (alpha x r): M(q, j) = B[q + alpha j];
            // an identity basis (a full-rank node) only splits the mode
            const DT& core = h.core(n.id);
            const bool ident = core.buf->identity && core.offset == 0 && b.alpha == b.r;
            DT next = ident ? cur : mode_mul(c, cur, static_cast<int>(pos), b.p, b.alpha, 1, b.alpha);
            const Shape& cs = core.shape;
            Shape sh = next.shape;
            sh[pos] = cs[0];
            sh.insert(sh.begin() + static_cast<std::ptrdiff_t>(pos) + 1, cs[1]);
            next.shape = sh;
            cur = next;
            modes[pos] = n.successors[0];
            modes.insert(modes.begin() + static_cast<std::ptrdiff_t>(pos) + 1, n.successors[1]);
            split = true;
            break;
        }
    }
    // validate() forces in-order spans: mode k now carries leaf dimension k
    for (size_t k = 0; k < modes.size(); ++k)
        if (h.tree.node(modes[k]).leaf_dim != static_cast<Index>(k)) raise(HTR_ERR_RUNTIME, "decode: unexpected mode order");
    // Leaves 0 and 1 last, in one fused kernel (k_decode.cu), when their
    // extents and ranks fit it: the other leaves expand first, then every
    // slab of the remaining modes and samples is reconstructed without an
    // intermediate.
    const Basis l0 = basis_of(h, modes[0]);
    const Basis l1 = modes.size() >= 2 ? basis_of(h, modes[1]) : l0;
    const bool fuse2 = c.fused && modes.size() >= 2 && cur.shape[0] == l0.r && cur.shape[1] == l1.r &&
                       decode2_supported(l0.alpha, l1.alpha, l0.r, l1.r) &&
                       (reinterpret_cast<uintptr_t>(dst) & 15u) == 0 &&
                       (!ref || (reinterpret_cast<uintptr_t>(ref->data()) & 15u) == 0);
    std::vector<size_t> order;
    for (size_t k = fuse2 ? 2 : 0; k < modes.size(); ++k) order.push_back(k);
    auto growth = [&](size_t k) {
        const Basis b = basis_of(h, modes[k]);
        return static_cast<double>(b.alpha) / static_cast<double>(std::max<int64_t>(b.r, 1));
    };
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return growth(a) < growth(b); });
    for (size_t i = 0; i < order.size(); ++i) {
        const size_t k = order[i];
        const Basis b = basis_of(h, modes[k]);
        cur = mode_mul(c, cur, static_cast<int>(k), b.p, b.alpha, 1, b.alpha,
                       !fuse2 && i + 1 == order.size() ? dst : nullptr);
    }
    if (fuse2) {
        Shape os = cur.shape;
        os[0] = l0.alpha;
        os[1] = l1.alpha;
        DT out;
        if (ref) {
            out.shape = os;
        } else if (dst) {
            out.shape = os;
            out.buf = std::make_shared<Buf>(c.st, dst, htrise::shape_product(os));
        } else {
            out = c.tensor(os);
        }
        Decode2Args a;
        a.W = cur.data();
        a.T = htrise::shape_product(cur.shape) / (l0.r * l1.r);
        a.r0 = static_cast<int>(l0.r);
        a.r1 = static_cast<int>(l1.r);
        a.n0 = l0.alpha;
        a.n1 = l1.alpha;
        a.U0 = l0.p;
        a.U1 = l1.p;
        BufPtr parts;
        if (ref) {
            a.X = nullptr;
            a.Y = ref->data();
            parts = c.alloc(decode2_partials(a.T, c.num_sms));
            a.partials = parts->p;
            // the kernel's last CTA sums the partials (and mirrors the total
            // into mapped host memory when asked)
            a.final_out = resid_out;
            a.final_host = resid_host;
            a.ticket = c.d_ticket;
        } else {
            a.X = out.data();
        }
        if (a.T > 0) {
            if (launch_decode2(a, c.num_sms, c.s, &c.launches) < 0) raise(HTR_ERR_RUNTIME, "decode: fused leaf kernel rejected its operands");
            HTR_CUDA(cudaGetLastError());
            if (ref && host_written) *host_written = resid_host != nullptr;
        } else if (ref) {
            HTR_CUDA(cudaMemsetAsync(resid_out, 0, sizeof(double), c.s));
        }
        return out;
    }
    if (ref) {
        const int64_t n = cur.size();
        BufPtr parts = c.alloc(std::max<int64_t>(1, 4 * c.num_sms));
        if (n > 0) {
            const int nb = launch_diff_sumsq(cur.data(), ref->data(), n, parts->p, c.num_sms, c.s, &c.launches);
            launch_sum_partials(parts->p, nb, resid_out, c.s, &c.launches);
        } else {
            HTR_CUDA(cudaMemsetAsync(resid_out, 0, sizeof(double), c.s));
        }
        HTR_CUDA(cudaGetLastError());
    }
    return cur;
}

}  // namespace

}  // namespace htr
