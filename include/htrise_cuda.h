/* htrise-b200 C-ABI: the drop-in boundary beneath the htrise C++ API.
 *
 * The reference (/root/reference/proj/include/htrise/ headers) is header-only
 * C++ with no plugin or FFI layer; its public entry points
 * are inline functions in namespace htrise. This library re-implements the
 * data-parallel core of those entry points as sm_100a kernels and exports it
 * through plain C symbols (no C++ or torch types) so that the C++ headers in
 * include/htrise/, a ctypes binding (paper_2412_16544_b200/htrise.py) or any
 * other FFI can bind it. Each function below names the reference interface it
 * replaces.
 *
 * Conventions
 *  - Every function returns an htr_status; HTR_OK == 0. On error the context's
 *    last-error string carries the message (same wording as the reference's
 *    exception text where one exists). Status codes map onto the reference's
 *    exception types: INVALID_ARGUMENT -> std::invalid_argument,
 *    OUT_OF_RANGE -> std::out_of_range, RUNTIME -> std::runtime_error.
 *  - Tensors are f64 in canonical order (first index fastest, reference
 *    tensor.hpp:36-41). Pointers flagged *_on_device are CUDA device pointers
 *    on the context's device; otherwise host pointers (pinned or pageable).
 *  - Representations (htr_rep) are device-resident values: non-root cores are
 *    immutable and shared; the root is an append-only device buffer with
 *    capacity. An update returns a NEW htr_rep and leaves its input valid
 *    (reference value semantics, ht_rise.hpp:99-101), in O(batch) for a skip.
 *  - One CUDA stream per context; thread-compatible, not thread-safe.
 */
#ifndef HTRISE_CUDA_H
#define HTRISE_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define HTR_API __attribute__((visibility("default")))
#else
#define HTR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t htr_status;
#define HTR_OK 0
#define HTR_ERR_INVALID_ARGUMENT 1
#define HTR_ERR_OUT_OF_RANGE 2
#define HTR_ERR_RUNTIME 3
#define HTR_ERR_CUDA 4
#define HTR_ERR_NO_DEVICE 5

#define HTR_MAX_NODES 256
#define HTR_MAX_LAYERS 16

/* NodeKind order of dimension_tree.hpp:14 */
#define HTR_KIND_ROOT 0
#define HTR_KIND_TRANSFER 1
#define HTR_KIND_LEAF 2

typedef struct htr_context htr_context;
typedef struct htr_rep htr_rep;

/* One TreeNode (dimension_tree.hpp:28-34); succ0/succ1 are positions in
 * layer+1 (-1 for leaves), leaf_dim is -1 for internal nodes. */
typedef struct {
    int32_t layer, pos, kind, leaf_dim, succ0, succ1;
} htr_node;

/* BuildReport (bht.hpp:170-174). */
typedef struct {
    double eps_nw_initial;
    int32_t n_records;
    int32_t rec_layer[HTR_MAX_NODES];
    int32_t rec_pos[HTR_MAX_NODES];
    int64_t rec_rank[HTR_MAX_NODES];
    double rec_discarded[HTR_MAX_NODES];
    int32_t n_layer_norms;
    double layer_norms[HTR_MAX_LAYERS];
} htr_build_report;

/* UpdateReport (ht_rise.hpp:20-27); per-node arrays in tree order
 * (layer 1..depth, position order). */
typedef struct {
    int32_t skipped;
    double proj_error;
    double eps_des;
    double seconds;
    int32_t n_nodes;
    int32_t node_layer[HTR_MAX_NODES];
    int32_t node_pos[HTR_MAX_NODES];
    int64_t added_ranks[HTR_MAX_NODES];
    int64_t new_ranks[HTR_MAX_NODES];
    /* device-side accounting of the call (not in the reference report) */
    int32_t used_fused_path;
    int32_t used_exact_loss;
    int64_t kernel_launches;
} htr_update_report;

/* ---- context -------------------------------------------------------- */
/* On failure *out is still set (a handle without a device) so that
 * htr_last_error() can report why; destroy it with htr_context_destroy(). */
HTR_API htr_status htr_context_create(int32_t device, htr_context** out);
HTR_API htr_status htr_context_destroy(htr_context* ctx);
HTR_API const char* htr_last_error(const htr_context* ctx);
/* CUDA stream the context launches on (cudaStream_t). */
HTR_API htr_status htr_context_stream(htr_context* ctx, void** stream);
/* Make the context's stream wait for all work already enqueued on `stream`
 * (e.g. torch's current stream that produced a device input). */
HTR_API htr_status htr_context_wait_stream(htr_context* ctx, void* stream);
HTR_API htr_status htr_synchronize(htr_context* ctx);
/* Options: see HTR_OPT_*. */
#define HTR_OPT_EXACT_LOSS 1      /* 1: per-step explicit residual loss like bht.hpp:357-365 (default 0 = telescoped with guard band) */
#define HTR_OPT_FUSED_ENCODE 2    /* 1 (default): fused DMMA leaf-projection kernel where it applies */
#define HTR_OPT_PROFILE_EVENTS 3  /* 1: record per-kernel CUDA events for the bench */
#define HTR_OPT_TAIL_KERNEL 4     /* skip-path tail of (1,(2,3)) trees: 0 auto (default: one sample per CTA, split over a cluster for small batches; the unit-dealt TMA kernel when the transfer basis is the identity), 1 one sample per CTA, 2 sample pairs */
#define HTR_OPT_EIG_SOLVER 5      /* truncation eigensolver: 1 (default) Householder tridiagonal + bisection + inverse iteration, 0 Jacobi */
HTR_API htr_status htr_context_set_option(htr_context* ctx, int32_t option, double value);
/* Kernel launches issued on this context so far (monotonic counter). */
HTR_API int64_t htr_context_launch_count(const htr_context* ctx);
/* Average duration (ms) of the fused encode kernel over calls since the last
 * reset, measured with CUDA events on the launching stream. */
HTR_API htr_status htr_context_kernel_timing(htr_context* ctx, double* fused_ms_total, int64_t* fused_calls,
                                     double* gemm_ms_total, int64_t* gemm_calls);
HTR_API htr_status htr_context_reset_timing(htr_context* ctx);

/* Multi-GPU: batch-axis sharding. Every rank passes the same 128-byte NCCL
 * unique id; afterwards norms and Gram partial sums are all-reduced over
 * NCCL (dlopen'd libnccl.so.2) and every rank holds its own batch shard. */
HTR_API htr_status htr_comm_get_unique_id(uint8_t out[128]);
HTR_API htr_status htr_context_init_comm(htr_context* ctx, const uint8_t unique_id[128], int32_t nranks,
                                 int32_t rank);

/* Host-staged alternative to NCCL: `fn` sums n doubles in place over all
 * ranks (element-wise, the same bits on every rank) and returns 0. The
 * library drains its stream, hands the partial sums to `fn` in pinned host
 * memory and copies the result back, so ranks never wait on one another's
 * kernels. For transports without NCCL peers (several ranks' processes on one
 * device in tests, a CPU transport such as gloo); the runtime path above the
 * reduction is the same as with NCCL. Every rank installs a reducer with the
 * same nranks. */
typedef int32_t (*htr_host_reduce_fn)(double* buf, int64_t n, void* user);
HTR_API htr_status htr_context_set_reducer(htr_context* ctx, htr_host_reduce_fn fn, void* user, int32_t nranks,
                                           int32_t rank);

/* ---- trees (dimension_tree.hpp) ------------------------------------- */
/* DimensionTree::balanced(d) (dimension_tree.hpp:44-94); writes 2d-1 nodes. */
HTR_API htr_status htr_tree_balanced(int64_t d, htr_node* out_nodes, int64_t capacity, int64_t* n_nodes,
                             char* err, int64_t err_len);
/* DimensionTree::from_layers validation (dimension_tree.hpp:99-113,170-250). */
HTR_API htr_status htr_tree_validate(const htr_node* nodes, int64_t n_nodes, char* err, int64_t err_len);

/* ---- BHT-l2r (bht.hpp:251-350) -------------------------------------- */
HTR_API htr_status htr_bht_l2r(htr_context* ctx, const double* y, int32_t y_on_device, const int64_t* shape,
                       int32_t order, const htr_node* nodes, int64_t n_nodes, double eps_rel,
                       int32_t adaptive_budget, htr_rep** out, htr_build_report* report);

/* ---- HT-RISE (ht_rise.hpp:99-186) ------------------------------------ */
/* eps_rel_override < 0 means "use the representation's own epsilon". */
HTR_API htr_status htr_ht_rise_update(htr_context* ctx, const htr_rep* in, const double* y, int32_t y_on_device,
                              const int64_t* shape, int32_t order, double eps_rel_override,
                              int32_t adaptive_budget, htr_rep** out, htr_update_report* report);

/* A stream of n updates (extension; the reference's caller loops
 * ht_rise_update over batches, tools/main.cpp:225-243): identical to n
 * htr_ht_rise_update calls each applied to the previous result, with the
 * skip-path encode of batch i+1 queued on the device before batch i's skip
 * decision is read back (a skip leaves the bases unchanged; after an
 * expansion the speculative work is discarded and batch i+1 re-runs).
 * ys[i] is batch i (all on the device or all on the host), shapes holds
 * n * order extents. On success outs[i] / reports[i] hold the value and the
 * report after batch i (free each value with htr_rep_free); on failure no
 * output is set. */
HTR_API htr_status htr_ht_rise_update_many(htr_context* ctx, const htr_rep* in, int64_t n, const double* const* ys,
                                   int32_t y_on_device, const int64_t* shapes, int32_t order,
                                   double eps_rel_override, int32_t adaptive_budget, htr_rep** outs,
                                   htr_update_report* reports);

/* ---- encode / decode / reconstruct (bht.hpp:373-479) ----------------- */
/* latent is r11 x r12 x N (canonical). */
HTR_API htr_status htr_encode(htr_context* ctx, const htr_rep* rep, const double* y, int32_t y_on_device,
                      const int64_t* shape, int32_t order, double* latent, int32_t latent_on_device,
                      double* proj_error);
HTR_API htr_status htr_decode(htr_context* ctx, const htr_rep* rep, const double* latent,
                      int32_t latent_on_device, const int64_t* latent_shape, double* out,
                      int32_t out_on_device);
/* m is 1-based (bht.hpp:472-479); out has prod(dims) entries. */
HTR_API htr_status htr_reconstruct_slice(htr_context* ctx, const htr_rep* rep, int64_t m, double* out,
                                 int32_t out_on_device);

/* Relative reconstruction error of one test tensor, the summand of
 * relative_test_error (metrics.hpp:218-237): ||y - decode(encode(y))|| / ||y||
 * (0 when ||y|| = 0). y is prod(dims) x N (order d + 1) or one sample
 * (order d). The reconstruction is compared on the device and, where the
 * fused decode kernel applies, never materialised. */
HTR_API htr_status htr_relative_error(htr_context* ctx, const htr_rep* rep, const double* y, int32_t y_on_device,
                              const int64_t* shape, int32_t order, double* rel_error);

/* ---- representation values ------------------------------------------ */
HTR_API htr_status htr_rep_free(htr_rep* rep);
HTR_API htr_status htr_rep_clone(htr_context* ctx, const htr_rep* rep, htr_rep** out);
HTR_API htr_status htr_rep_info(const htr_rep* rep, int32_t* d, int64_t* dims, int64_t* accumulated,
                        double* epsilon_rel, int64_t* n_nodes);
/* Samples held by this value: `local` slices in this rank's root shard and
 * `global` streamed over all ranks (equal on an unsharded context;
 * htr_rep_info's `accumulated` is the global count). */
HTR_API htr_status htr_rep_counts(const htr_rep* rep, int64_t* local, int64_t* global);
HTR_API htr_status htr_rep_nodes(const htr_rep* rep, htr_node* nodes, int64_t capacity);
/* Core shape (2 entries for leaves, 3 otherwise; the root's last extent is
 * the LOCAL sample count on a sharded context). */
HTR_API htr_status htr_rep_core_shape(const htr_rep* rep, int32_t layer, int32_t pos, int64_t* shape,
                              int32_t* order);
HTR_API htr_status htr_rep_core_get(htr_context* ctx, const htr_rep* rep, int32_t layer, int32_t pos,
                            double* out, int32_t out_on_device);
/* Build a representation from host cores given in tree order (layer 0..p,
 * position order; root first). */
HTR_API htr_status htr_rep_import(htr_context* ctx, const htr_node* nodes, int64_t n_nodes, const int64_t* dims,
                          int32_t d, const double* const* cores, const int64_t* core_shapes /* 3 per node */,
                          int64_t accumulated, double eps_rel, htr_rep** out);
/* Reserve root capacity (in samples) so that later appends never reallocate. */
HTR_API htr_status htr_rep_reserve(htr_context* ctx, htr_rep* rep, int64_t samples);

/* ---- building blocks (truncated_svd.hpp, tensor.hpp, ht_rise.hpp) ----- */
/* truncated_svd (truncated_svd.hpp:53-100) of a rows x cols matrix; u gets
 * rows x rank (capacity rows*min(rows,cols)), sigma gets rank values. */
HTR_API htr_status htr_truncated_svd(htr_context* ctx, const double* m, int32_t m_on_device, int64_t rows,
                             int64_t cols, double eps_abs, int64_t min_rank, double* u, double* sigma,
                             int64_t* rank, double* discarded_norm);
/* mode_multiply (tensor.hpp:300-312): out = t x_mode M, M is q x extent
 * (column-major) and lives where t lives (t_on_device). */
HTR_API htr_status htr_mode_multiply(htr_context* ctx, const double* t, int32_t t_on_device, const int64_t* shape,
                             int32_t order, int32_t mode, const double* m, int64_t q, double* out,
                             int32_t out_on_device);
/* Dense products of the tensor algebra (reference tensor.hpp, Eigen's GEMM
 * in the reference), host buffers in and out, computed on the device:
 *  htr_matmul:       C (m x n) = A (m x k) B (k x n), column-major
 *                    (Matrix::operator*, the GEMM behind unfold-based products);
 *  htr_contract:     contract(a, da, b, db) (tensor.hpp:273-296): out is
 *                    a's remaining modes then b's, canonical;
 *  htr_permute_axes: permute_axes (tensor.hpp:219-267): output mode k is
 *                    input mode perm[k] (order <= 16). */
HTR_API htr_status htr_matmul(htr_context* ctx, const double* a, int64_t m, int64_t k, const double* b, int64_t n,
                              double* c);
HTR_API htr_status htr_contract(htr_context* ctx, const double* a, const int64_t* a_shape, int32_t a_order, int32_t da,
                                const double* b, const int64_t* b_shape, int32_t b_order, int32_t db, double* out);
HTR_API htr_status htr_permute_axes(htr_context* ctx, const double* t, const int64_t* shape, int32_t order,
                                    const int64_t* perm, double* out);
/* Device memory for batches the caller keeps on the device (e.g. ingested
 * and normalised there before compression): cudaMalloc'd on the context's
 * device; htr_copy moves n doubles between host and device buffers. */
HTR_API htr_status htr_device_alloc(htr_context* ctx, int64_t n, double** ptr);
HTR_API htr_status htr_device_free(htr_context* ctx, double* ptr);
HTR_API htr_status htr_copy(htr_context* ctx, double* dst, int32_t dst_on_device, const double* src,
                            int32_t src_on_device, int64_t n);

/* normalize (metrics.hpp:93-171) on the device: method 0 none, 1 maxabs,
 * 2 unitvec, 3 zscore (population sigma); field_axis -1 for one field, else
 * one field per slice along that mode. scale / offset / floored receive one
 * entry per field (zero scales floored to 1); out receives the scaled tensor
 * (out may equal y on the device: in place). The per-field maxima are exact;
 * sums are deterministic tree reductions (the reference sums sequentially:
 * the recorded scales may differ in the last bit). */
HTR_API htr_status htr_normalize(htr_context* ctx, const double* y, int32_t y_on_device, const int64_t* shape,
                                 int32_t order, int32_t method, int32_t field_axis, double* out,
                                 int32_t out_on_device, double* scale, double* offset, int32_t* floored);
/* denormalize (metrics.hpp:174-197): out = y * scale[f] + offset[f]. */
HTR_API htr_status htr_denormalize(htr_context* ctx, const double* y, int32_t y_on_device, const int64_t* shape,
                                   int32_t order, int32_t method, int32_t field_axis, const double* scale,
                                   const double* offset, double* out, int32_t out_on_device);

/* compute_residual (ht_rise.hpp:31-38): R = C - U (U^T C). */
HTR_API htr_status htr_compute_residual(htr_context* ctx, const double* u, int64_t rows, int64_t r, const double* c,
                                int64_t cols, double* out);
/* frobenius_norm (tensor.hpp:269) of n doubles. */
HTR_API htr_status htr_frobenius_norm(htr_context* ctx, const double* t, int32_t t_on_device, int64_t n,
                              double* out);

#ifdef __cplusplus
}
#endif

#endif /* HTRISE_CUDA_H */
