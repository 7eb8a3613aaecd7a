// extern "C" boundary (include/htrise_cuda.h): status codes instead of
// exceptions, plain pointers instead of C++ types.
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>

#include "runtime.hpp"

struct htr_context {
    std::unique_ptr<htr::Context> ctx;
    std::string err;
};

struct htr_rep {
    std::shared_ptr<htr::Rep> rep;
};

namespace htr {
void comm_unique_id(uint8_t out[128]);
void comm_init(Context& c, const uint8_t uid[128], int nranks, int rank);
void set_reducer(Context& c, htr_host_reduce_fn fn, void* user, int nranks, int rank);
}  // namespace htr

namespace {

using htr::BufPtr;
using htr::DT;
using htr::Shape;

template <typename F>
htr_status guarded(htr_context* c, F&& f) {
    try {
        f();
        return HTR_OK;
    } catch (const htr::Error& e) {
        if (c) c->err = e.msg;
        return e.code;
    } catch (const std::invalid_argument& e) {
        if (c) c->err = e.what();
        return HTR_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        if (c) c->err = e.what();
        return HTR_ERR_OUT_OF_RANGE;
    } catch (const std::exception& e) {
        if (c) c->err = e.what();
        return HTR_ERR_RUNTIME;
    }
}

void copy_err(const std::string& m, char* err, int64_t len) {
    if (err && len > 0) {
        std::strncpy(err, m.c_str(), static_cast<size_t>(len - 1));
        err[len - 1] = '\0';
    }
}

template <typename F>
htr_status guarded_noctx(char* err, int64_t len, F&& f) {
    try {
        f();
        return HTR_OK;
    } catch (const htr::Error& e) {
        copy_err(e.msg, err, len);
        return e.code;
    } catch (const std::invalid_argument& e) {
        copy_err(e.what(), err, len);
        return HTR_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        copy_err(e.what(), err, len);
        return HTR_ERR_OUT_OF_RANGE;
    } catch (const std::exception& e) {
        copy_err(e.what(), err, len);
        return HTR_ERR_RUNTIME;
    }
}

htr::Context& C(htr_context* c) {
    if (!c || !c->ctx) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null context");
    // every entry point runs on the context's device, whatever device the
    // caller (torch, another library) made current
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != c->ctx->device) HTR_CUDA(cudaSetDevice(c->ctx->device));
    return *c->ctx;
}

Shape to_shape(const int64_t* shape, int32_t order) {
    if (!shape || order < 1) htr::raise(HTR_ERR_INVALID_ARGUMENT, "DenseTensor: empty shape");
    Shape s(shape, shape + order);
    for (int64_t e : s)
        if (e < 1) htr::raise(HTR_ERR_INVALID_ARGUMENT, "DenseTensor: extent " + std::to_string(e) + " < 1");
    return s;
}

/// Wrap (device) or upload (host) an input tensor.
DT input(htr::Context& c, const double* p, bool on_device, const Shape& shape) {
    DT t;
    t.shape = shape;
    const int64_t n = htrise::shape_product(shape);
    if (!p) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null tensor pointer");
    if (on_device) {
        t.buf = std::make_shared<htr::Buf>(c.st, const_cast<double*>(p), n);
    } else {
        t.buf = c.alloc(n);
        HTR_CUDA(cudaMemcpyAsync(t.buf->p, p, sizeof(double) * static_cast<size_t>(n), cudaMemcpyHostToDevice, c.s));
    }
    return t;
}

void output(htr::Context& c, const double* src, int64_t n, double* dst, bool on_device) {
    if (n == 0) return;
    if (!dst) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null output pointer");
    HTR_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * static_cast<size_t>(n),
                             on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.s));
    HTR_CUDA(cudaStreamSynchronize(c.s));
}

const htr::Rep& R(const htr_rep* r) {
    if (!r || !r->rep) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null representation");
    return *r->rep;
}

}  // namespace

extern "C" {

htr_status htr_context_create(int32_t device, htr_context** out) {
    if (!out) return HTR_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    auto* c = new htr_context;
    htr_status st = guarded(c, [&] { c->ctx = std::make_unique<htr::Context>(device); });
    // on failure the handle is still returned (without a device context) so
    // the caller can read htr_last_error() before htr_context_destroy()
    *out = c;
    return st;
}

htr_status htr_context_destroy(htr_context* ctx) {
    delete ctx;
    return HTR_OK;
}

const char* htr_last_error(const htr_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

htr_status htr_context_stream(htr_context* ctx, void** stream) {
    return guarded(ctx, [&] { *stream = C(ctx).s; });
}

htr_status htr_context_wait_stream(htr_context* ctx, void* stream) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        HTR_CUDA(cudaEventRecord(c.ev[3], static_cast<cudaStream_t>(stream)));
        HTR_CUDA(cudaStreamWaitEvent(c.s, c.ev[3], 0));
    });
}

htr_status htr_synchronize(htr_context* ctx) {
    return guarded(ctx, [&] { HTR_CUDA(cudaStreamSynchronize(C(ctx).s)); });
}

htr_status htr_context_set_option(htr_context* ctx, int32_t option, double value) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        switch (option) {
            case HTR_OPT_EXACT_LOSS: c.exact_loss = value != 0.0; break;
            case HTR_OPT_FUSED_ENCODE: c.fused = value != 0.0; break;
            case HTR_OPT_PROFILE_EVENTS: c.profile = value != 0.0; break;
            case HTR_OPT_TAIL_KERNEL:
                if (value < 0 || value > 2) htr::raise(HTR_ERR_INVALID_ARGUMENT, "tail kernel option: 0, 1 or 2");
                c.tail_kernel = static_cast<int>(value);
                break;
            case HTR_OPT_EIG_SOLVER: c.tridiag = value != 0.0; break;
            default: htr::raise(HTR_ERR_INVALID_ARGUMENT, "unknown option " + std::to_string(option));
        }
    });
}

int64_t htr_context_launch_count(const htr_context* ctx) { return ctx && ctx->ctx ? ctx->ctx->launches : -1; }

htr_status htr_context_kernel_timing(htr_context* ctx, double* fused_ms_total, int64_t* fused_calls,
                                     double* gemm_ms_total, int64_t* gemm_calls) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (fused_ms_total) *fused_ms_total = c.fused_ms;
        if (fused_calls) *fused_calls = c.fused_calls;
        if (gemm_ms_total) *gemm_ms_total = c.gemm_ms;
        if (gemm_calls) *gemm_calls = c.gemm_calls;
    });
}

htr_status htr_context_reset_timing(htr_context* ctx) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        c.fused_ms = c.gemm_ms = 0.0;
        c.fused_calls = c.gemm_calls = 0;
    });
}

htr_status htr_comm_get_unique_id(uint8_t out[128]) {
    return guarded_noctx(nullptr, 0, [&] { htr::comm_unique_id(out); });
}

htr_status htr_context_init_comm(htr_context* ctx, const uint8_t unique_id[128], int32_t nranks, int32_t rank) {
    return guarded(ctx, [&] { htr::comm_init(C(ctx), unique_id, nranks, rank); });
}

htr_status htr_context_set_reducer(htr_context* ctx, htr_host_reduce_fn fn, void* user, int32_t nranks, int32_t rank) {
    return guarded(ctx, [&] { htr::set_reducer(C(ctx), fn, user, nranks, rank); });
}

htr_status htr_tree_balanced(int64_t d, htr_node* out_nodes, int64_t capacity, int64_t* n_nodes, char* err,
                             int64_t err_len) {
    return guarded_noctx(err, err_len, [&] {
        htrise::DimensionTree t = htrise::DimensionTree::balanced(d);
        std::vector<htr_node> nodes;
        htr::nodes_from_tree(t, nodes);
        if (n_nodes) *n_nodes = static_cast<int64_t>(nodes.size());
        if (static_cast<int64_t>(nodes.size()) > capacity) htr::raise(HTR_ERR_OUT_OF_RANGE, "node buffer too small");
        std::memcpy(out_nodes, nodes.data(), nodes.size() * sizeof(htr_node));
    });
}

htr_status htr_tree_validate(const htr_node* nodes, int64_t n_nodes, char* err, int64_t err_len) {
    return guarded_noctx(err, err_len, [&] { (void)htr::tree_from_nodes(nodes, n_nodes); });
}

htr_status htr_bht_l2r(htr_context* ctx, const double* y, int32_t y_on_device, const int64_t* shape, int32_t order,
                       const htr_node* nodes, int64_t n_nodes, double eps_rel, int32_t adaptive_budget, htr_rep** out,
                       htr_build_report* report) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        htrise::DimensionTree tree = htr::tree_from_nodes(nodes, n_nodes);
        Shape s = to_shape(shape, order);
        htr::check_batch_input(s, tree, nullptr, "bht_l2r");
        DT yt = input(c, y, y_on_device != 0, s);
        htr::BuildOut b = htr::bht_l2r(c, yt, tree, eps_rel, adaptive_budget != 0);
        HTR_CUDA(cudaStreamSynchronize(c.s));
        if (report) *report = b.report;
        *out = new htr_rep{b.rep};
    });
}

htr_status htr_ht_rise_update(htr_context* ctx, const htr_rep* in, const double* y, int32_t y_on_device,
                              const int64_t* shape, int32_t order, double eps_rel_override, int32_t adaptive_budget,
                              htr_rep** out, htr_update_report* report) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        const htr::Rep& h = R(in);
        Shape s = to_shape(shape, order);
        htr::check_batch_input(s, h.tree, &h.dims, "ht_rise_update");
        DT yt = input(c, y, y_on_device != 0, s);
        htr::UpdateOut u = htr::ht_rise_update(c, h, yt, eps_rel_override, adaptive_budget != 0);
        if (report) *report = u.report;
        *out = new htr_rep{u.rep};
    });
}

htr_status htr_ht_rise_update_many(htr_context* ctx, const htr_rep* in, int64_t n, const double* const* ys,
                                   int32_t y_on_device, const int64_t* shapes, int32_t order, double eps_rel_override,
                                   int32_t adaptive_budget, htr_rep** outs, htr_update_report* reports) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (n < 0) htr::raise(HTR_ERR_INVALID_ARGUMENT, "ht_rise_update_many: negative batch count");
        if (n > 0 && (!ys || !shapes || !outs)) htr::raise(HTR_ERR_INVALID_ARGUMENT, "ht_rise_update_many: null argument");
        auto batch_of = [&](int64_t i) {
            Shape s = to_shape(shapes + i * order, order);
            return input(c, ys[i], y_on_device != 0, s);
        };
        (void)R(in);
        std::vector<htr::UpdateOut> us =
            htr::ht_rise_update_many(c, in->rep, n, batch_of, eps_rel_override, adaptive_budget != 0);
        for (int64_t i = 0; i < n; ++i) {
            if (reports) reports[i] = us[static_cast<size_t>(i)].report;
            outs[i] = new htr_rep{us[static_cast<size_t>(i)].rep};
        }
    });
}

htr_status htr_encode(htr_context* ctx, const htr_rep* rep, const double* y, int32_t y_on_device, const int64_t* shape,
                      int32_t order, double* latent, int32_t latent_on_device, double* proj_error) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        const htr::Rep& h = R(rep);
        Shape s = to_shape(shape, order);
        htr::check_batch_input(s, h.tree, &h.dims, "encode");
        DT yt = input(c, y, y_on_device != 0, s);
        htr::EncodeOut e = htr::encode(c, h, yt, c.exact_loss);
        if (e.nonfinite) htr::raise(HTR_ERR_INVALID_ARGUMENT, "encode: non-finite input");
        if (proj_error) *proj_error = std::sqrt(e.proj_sq);
        if (latent) output(c, e.latent.data(), e.latent.size(), latent, latent_on_device != 0);
        HTR_CUDA(cudaStreamSynchronize(c.s));
    });
}

htr_status htr_decode(htr_context* ctx, const htr_rep* rep, const double* latent, int32_t latent_on_device,
                      const int64_t* latent_shape, double* out, int32_t out_on_device) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        const htr::Rep& h = R(rep);
        Shape s = to_shape(latent_shape, 3);
        DT lt = input(c, latent, latent_on_device != 0, s);
        if (out_on_device) {  // straight into the caller's buffer
            if (!out) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null output pointer");
            htr::decode(c, h, lt, out);
            HTR_CUDA(cudaStreamSynchronize(c.s));
            return;
        }
        DT full = htr::decode(c, h, lt);
        output(c, full.data(), full.size(), out, false);
    });
}

htr_status htr_reconstruct_slice(htr_context* ctx, const htr_rep* rep, int64_t m, double* out, int32_t out_on_device) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        const htr::Rep& h = R(rep);
        if (m < 1 || m > h.acc)
            htr::raise(HTR_ERR_OUT_OF_RANGE,
                       "reconstruct_slice: index " + std::to_string(m) + " outside 1.." + std::to_string(h.acc));
        DT lt;
        lt.buf = h.root->buf;
        lt.offset = h.root->r11 * h.root->r12 * (m - 1);
        lt.shape = {h.root->r11, h.root->r12, 1};
        if (out_on_device) {
            if (!out) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null output pointer");
            htr::decode(c, h, lt, out);
            HTR_CUDA(cudaStreamSynchronize(c.s));
            return;
        }
        DT full = htr::decode(c, h, lt);
        output(c, full.data(), full.size(), out, false);
    });
}

htr_status htr_relative_error(htr_context* ctx, const htr_rep* rep, const double* y, int32_t y_on_device,
                              const int64_t* shape, int32_t order, double* rel_error) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        const htr::Rep& h = R(rep);
        if (!rel_error) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null output pointer");
        Shape s = to_shape(shape, order);
        if (static_cast<htrise::Index>(s.size()) == h.tree.dims()) s.push_back(1);  // metrics.hpp:224-226
        htr::check_batch_input(s, h.tree, &h.dims, "encode");  // the reference fails inside encode
        DT yt = input(c, y, y_on_device != 0, s);
        htr::EncodeOut e = htr::encode(c, h, yt, false);
        if (e.nonfinite) htr::raise(HTR_ERR_INVALID_ARGUMENT, "encode: non-finite input");
        htr::BufPtr r = c.alloc(1);
        htr::decode_residual_sq(c, h, e.latent, yt, r->p);
        c.allreduce(r->p, 1);
        double rsq = 0.0;
        c.fetch(r->p, 1, &rsq);
        *rel_error = e.ysq == 0.0 ? 0.0 : std::sqrt(rsq) / std::sqrt(e.ysq);
    });
}

htr_status htr_rep_free(htr_rep* rep) {
    delete rep;
    return HTR_OK;
}

htr_status htr_rep_clone(htr_context* ctx, const htr_rep* rep, htr_rep** out) {
    return guarded(ctx, [&] { *out = new htr_rep{std::make_shared<htr::Rep>(R(rep))}; });
}

htr_status htr_rep_info(const htr_rep* rep, int32_t* d, int64_t* dims, int64_t* accumulated, double* epsilon_rel,
                        int64_t* n_nodes) {
    return guarded(nullptr, [&] {
        const htr::Rep& h = R(rep);
        if (d) *d = static_cast<int32_t>(h.tree.dims());
        if (dims)
            for (size_t k = 0; k < h.dims.size(); ++k) dims[k] = h.dims[k];
        if (accumulated) *accumulated = h.acc_global;
        if (epsilon_rel) *epsilon_rel = h.eps_rel;
        if (n_nodes) *n_nodes = 2 * h.tree.dims() - 1;
    });
}

htr_status htr_rep_counts(const htr_rep* rep, int64_t* local, int64_t* global) {
    return guarded(nullptr, [&] {
        const htr::Rep& h = R(rep);
        if (local) *local = h.acc;
        if (global) *global = h.acc_global;
    });
}

htr_status htr_rep_nodes(const htr_rep* rep, htr_node* nodes, int64_t capacity) {
    return guarded(nullptr, [&] {
        std::vector<htr_node> v;
        htr::nodes_from_tree(R(rep).tree, v);
        if (static_cast<int64_t>(v.size()) > capacity) htr::raise(HTR_ERR_OUT_OF_RANGE, "node buffer too small");
        std::memcpy(nodes, v.data(), v.size() * sizeof(htr_node));
    });
}

htr_status htr_rep_core_shape(const htr_rep* rep, int32_t layer, int32_t pos, int64_t* shape, int32_t* order) {
    return guarded(nullptr, [&] {
        const htr::Rep& h = R(rep);
        const htrise::TreeNode& n = h.tree.node({layer, pos});
        if (n.kind == htrise::NodeKind::Root) {
            shape[0] = h.root->r11;
            shape[1] = h.root->r12;
            shape[2] = h.acc;
            *order = 3;
            return;
        }
        const DT& c = h.core({layer, pos});
        for (size_t k = 0; k < c.shape.size(); ++k) shape[k] = c.shape[k];
        *order = static_cast<int32_t>(c.shape.size());
    });
}

htr_status htr_rep_core_get(htr_context* ctx, const htr_rep* rep, int32_t layer, int32_t pos, double* out,
                            int32_t out_on_device) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        const htr::Rep& h = R(rep);
        const htrise::TreeNode& n = h.tree.node({layer, pos});
        if (n.kind == htrise::NodeKind::Root) {
            output(c, h.root->buf->p, h.root->r11 * h.root->r12 * h.acc, out, out_on_device != 0);
        } else {
            const DT& t = h.core({layer, pos});
            output(c, t.data(), t.size(), out, out_on_device != 0);
        }
    });
}

htr_status htr_rep_import(htr_context* ctx, const htr_node* nodes, int64_t n_nodes, const int64_t* dims, int32_t d,
                          const double* const* cores, const int64_t* core_shapes, int64_t accumulated, double eps_rel,
                          htr_rep** out) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        auto h = std::make_shared<htr::Rep>();
        h->st = c.st;
        h->tree = htr::tree_from_nodes(nodes, n_nodes);
        if (d != h->tree.dims()) htr::raise(HTR_ERR_INVALID_ARGUMENT, "HTRepresentation: dims/tree mismatch");
        h->dims = Shape(dims, dims + d);
        h->eps_rel = eps_rel;
        h->cores.resize(static_cast<size_t>(h->tree.depth()) + 1);
        int64_t i = 0;
        for (htrise::Index l = 0; l <= h->tree.depth(); ++l) {
            h->cores[static_cast<size_t>(l)].resize(static_cast<size_t>(h->tree.layer_size(l)));
            for (const htrise::TreeNode& n : h->tree.layer(l)) {
                const int64_t* cs = core_shapes + 3 * i;
                if (n.kind == htrise::NodeKind::Root) {
                    h->root = std::make_shared<htr::RootStore>();
                    h->root->r11 = cs[0];
                    h->root->r12 = cs[1];
                    h->root->cap = std::max<int64_t>(cs[2], 1);
                    h->root->buf = c.alloc(cs[0] * cs[1] * h->root->cap);
                    HTR_CUDA(cudaMemcpyAsync(h->root->buf->p, cores[i], sizeof(double) * static_cast<size_t>(cs[0] * cs[1] * cs[2]),
                                             cudaMemcpyHostToDevice, c.s));
                    h->root->committed = cs[2];
                    h->acc = cs[2];
                } else {
                    Shape s = n.kind == htrise::NodeKind::Leaf ? Shape{cs[0], cs[1]} : Shape{cs[0], cs[1], cs[2]};
                    DT t = c.tensor(s);
                    HTR_CUDA(cudaMemcpyAsync(t.data(), cores[i], sizeof(double) * static_cast<size_t>(t.size()),
                                             cudaMemcpyHostToDevice, c.s));
                    h->cores[static_cast<size_t>(l)][static_cast<size_t>(n.id.pos)] = t;
                }
                ++i;
            }
        }
        h->acc_global = accumulated;
        htr::measure_defect(c, *h);
        HTR_CUDA(cudaStreamSynchronize(c.s));
        *out = new htr_rep{h};
    });
}

htr_status htr_rep_reserve(htr_context* ctx, htr_rep* rep, int64_t samples) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (!rep || !rep->rep) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null representation");
        htr::Rep& h = *rep->rep;
        auto& rs = h.root;
        if (samples <= rs->cap) return;
        auto ns = std::make_shared<htr::RootStore>();
        ns->r11 = rs->r11;
        ns->r12 = rs->r12;
        ns->cap = samples;
        ns->buf = c.alloc(ns->r11 * ns->r12 * samples);
        HTR_CUDA(cudaMemcpyAsync(ns->buf->p, rs->buf->p, sizeof(double) * static_cast<size_t>(rs->r11 * rs->r12 * h.acc),
                                 cudaMemcpyDeviceToDevice, c.s));
        ns->committed = h.acc;
        h.root = ns;
        HTR_CUDA(cudaStreamSynchronize(c.s));
    });
}

htr_status htr_truncated_svd(htr_context* ctx, const double* m, int32_t m_on_device, int64_t rows, int64_t cols,
                             double eps_abs, int64_t min_rank, double* u, double* sigma, int64_t* rank,
                             double* discarded_norm) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (rows < 1 || cols < 1) htr::raise(HTR_ERR_INVALID_ARGUMENT, "truncated_svd: empty matrix");
        if (!(eps_abs >= 0)) htr::raise(HTR_ERR_INVALID_ARGUMENT, "truncated_svd: negative tolerance");
        DT mt = input(c, m, m_on_device != 0, {rows, cols});
        double s2 = 0.0;
        bool bad = false;
        htr::norm_sq(c, mt.data(), mt.size(), &s2, &bad, false);
        if (bad) htr::raise(HTR_ERR_INVALID_ARGUMENT, "truncated_svd: non-finite entries");
        htr::Truncation t = htr::truncate_mode(c, mt, 0, nullptr, eps_abs, min_rank, cols, false);
        if (rank) *rank = t.rank;
        if (discarded_norm) *discarded_norm = t.discarded;
        if (sigma)
            for (int64_t i = 0; i < t.rank; ++i) sigma[i] = t.sigma[static_cast<size_t>(i)];
        if (u) output(c, t.u.data(), rows * t.rank, u, false);
    });
}

htr_status htr_mode_multiply(htr_context* ctx, const double* t, int32_t t_on_device, const int64_t* shape,
                             int32_t order, int32_t mode, const double* m, int64_t q, double* out,
                             int32_t out_on_device) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        Shape s = to_shape(shape, order);
        if (mode < 0 || mode >= order)
            htr::raise(HTR_ERR_INVALID_ARGUMENT, "mode_multiply: mode " + std::to_string(mode) +
                                                     " out of range for order " + std::to_string(order));
        DT tt = input(c, t, t_on_device != 0, s);
        const int64_t J = s[static_cast<size_t>(mode)];
        DT mt = input(c, m, t_on_device != 0, {q, J});
        DT o = htr::mode_mul(c, tt, mode, mt.data(), q, 1, q);
        output(c, o.data(), o.size(), out, out_on_device != 0);
    });
}

htr_status htr_matmul(htr_context* ctx, const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c_out) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (m < 0 || k < 0 || n < 0) htr::raise(HTR_ERR_INVALID_ARGUMENT, "Matrix: product shape mismatch");
        if (m == 0 || n == 0) return;
        if (k == 0) {
            std::memset(c_out, 0, sizeof(double) * static_cast<size_t>(m * n));
            return;
        }
        DT at = input(c, a, false, {m, k});
        DT bt = input(c, b, false, {k, n});
        DT ct = c.tensor({m, n});
        htr::GemmDesc d;
        d.M = m; d.N1 = n; d.K1 = k;
        d.A = at.data(); d.sam = 1; d.sak1 = m;
        d.B = bt.data(); d.sbk1 = 1; d.sbn1 = k;
        d.C = ct.data(); d.scm = 1; d.scn1 = m;
        htr::run_gemm(c, d);
        output(c, ct.data(), m * n, c_out, false);
    });
}

htr_status htr_contract(htr_context* ctx, const double* a, const int64_t* a_shape, int32_t a_order, int32_t da,
                        const double* b, const int64_t* b_shape, int32_t b_order, int32_t db, double* out) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        Shape sa = to_shape(a_shape, a_order), sb = to_shape(b_shape, b_order);
        if (da < 0 || da >= a_order || db < 0 || db >= b_order)
            htr::raise(HTR_ERR_INVALID_ARGUMENT, "contract: mode out of range");
        const int64_t K = sa[static_cast<size_t>(da)];
        if (K != sb[static_cast<size_t>(db)])
            htr::raise(HTR_ERR_INVALID_ARGUMENT, "contract: extent mismatch " + std::to_string(K) + " vs " +
                                                     std::to_string(sb[static_cast<size_t>(db)]));
        DT at = input(c, a, false, sa), bt = input(c, b, false, sb);
        auto unfold = [&](const DT& t, int mode) {
            int64_t inner = 1, outer = 1;
            for (int k = 0; k < mode; ++k) inner *= t.shape[static_cast<size_t>(k)];
            for (size_t k = static_cast<size_t>(mode) + 1; k < t.shape.size(); ++k) outer *= t.shape[k];
            DT u = c.tensor({t.shape[static_cast<size_t>(mode)], inner * outer});
            htr::launch_unfold(t.data(), inner, t.shape[static_cast<size_t>(mode)], outer, u.data(), c.s, &c.launches);
            HTR_CUDA(cudaGetLastError());
            return u;
        };
        DT ua = unfold(at, da), ub = unfold(bt, db);
        const int64_t ra = ua.shape[1], rb = ub.shape[1];
        DT ct = c.tensor({ra, rb});
        htr::GemmDesc d;  // C = A_(da)^T B_(db)
        d.M = ra; d.N1 = rb; d.K1 = K;
        d.A = ua.data(); d.sam = K; d.sak1 = 1;
        d.B = ub.data(); d.sbk1 = 1; d.sbn1 = K;
        d.C = ct.data(); d.scm = 1; d.scn1 = ra;
        htr::run_gemm(c, d);
        output(c, ct.data(), ra * rb, out, false);
    });
}

htr_status htr_permute_axes(htr_context* ctx, const double* t, const int64_t* shape, int32_t order, const int64_t* perm,
                            double* out) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        Shape s = to_shape(shape, order);
        if (order > 16) htr::raise(HTR_ERR_INVALID_ARGUMENT, "permute_axes: at most 16 modes");
        std::vector<char> used(static_cast<size_t>(order), 0);
        for (int32_t k = 0; k < order; ++k) {
            if (perm[k] < 0 || perm[k] >= order || used[static_cast<size_t>(perm[k])])
                htr::raise(HTR_ERR_INVALID_ARGUMENT, "permute_axes: invalid permutation");
            used[static_cast<size_t>(perm[k])] = 1;
        }
        DT tt = input(c, t, false, s);
        DT o = c.tensor(s);
        htr::launch_permute(tt.data(), s.data(), order, perm, o.data(), c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        output(c, o.data(), o.size(), out, false);
    });
}

htr_status htr_device_alloc(htr_context* ctx, int64_t n, double** ptr) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        (void)c;
        if (!ptr || n < 0) htr::raise(HTR_ERR_INVALID_ARGUMENT, "device_alloc: bad arguments");
        *ptr = nullptr;
        if (n > 0) HTR_CUDA(cudaMalloc(reinterpret_cast<void**>(ptr), static_cast<size_t>(n) * sizeof(double)));
    });
}

htr_status htr_device_free(htr_context* ctx, double* ptr) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (ptr) {
            HTR_CUDA(cudaStreamSynchronize(c.s));  // the context's work on it is done
            HTR_CUDA(cudaFree(ptr));
        }
    });
}

htr_status htr_copy(htr_context* ctx, double* dst, int32_t dst_on_device, const double* src, int32_t src_on_device,
                    int64_t n) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        if (n <= 0) return;
        if (!dst || !src) htr::raise(HTR_ERR_INVALID_ARGUMENT, "copy: null pointer");
        const cudaMemcpyKind kind = dst_on_device ? (src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice)
                                                  : (src_on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost);
        HTR_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * static_cast<size_t>(n), kind, c.s));
        HTR_CUDA(cudaStreamSynchronize(c.s));
    });
}

namespace {
/// (inner, fields) of the field view of a canonical tensor (metrics.hpp:60-74)
std::pair<int64_t, int> field_view(const Shape& s, int32_t field_axis, int32_t order) {
    if (field_axis < 0) return {htrise::shape_product(s), 1};
    if (field_axis >= order)
        htr::raise(HTR_ERR_INVALID_ARGUMENT, "normalize: mode " + std::to_string(field_axis) +
                                                 " out of range for order " + std::to_string(order));
    int64_t inner = 1;
    for (int32_t k = 0; k < field_axis; ++k) inner *= s[static_cast<size_t>(k)];
    return {inner, static_cast<int>(s[static_cast<size_t>(field_axis)])};
}
}  // namespace

htr_status htr_normalize(htr_context* ctx, const double* y, int32_t y_on_device, const int64_t* shape, int32_t order,
                         int32_t method, int32_t field_axis, double* out, int32_t out_on_device, double* scale,
                         double* offset, int32_t* floored) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        Shape s = to_shape(shape, order);
        if (method < 0 || method > 3) htr::raise(HTR_ERR_INVALID_ARGUMENT, "unknown normalization method");
        const auto [inner, F] = field_view(s, field_axis, order);
        const int64_t n = htrise::shape_product(s);
        DT yt = input(c, y, y_on_device != 0, s);
        std::vector<double> sc(static_cast<size_t>(F), method == 0 ? 1.0 : 0.0), mu(static_cast<size_t>(F), 0.0);
        std::vector<int32_t> fl(static_cast<size_t>(F), 0);
        BufPtr parts = c.alloc(static_cast<int64_t>(htr::field_stat_blocks(c.num_sms)) * 16);
        BufPtr stat = c.alloc(F), dmu = c.alloc(F), dsc = c.alloc(F);
        auto stat_of = [&](int kind, const double* mup) {
            htr::launch_field_stat(yt.data(), n, inner, F, kind, mup, parts->p, stat->p, c.num_sms, c.s, &c.launches);
            HTR_CUDA(cudaGetLastError());
            std::vector<double> v(static_cast<size_t>(F));
            c.fetch(stat->p, F, v.data());
            return v;
        };
        const double count = static_cast<double>(n / F);
        if (method == 1) {
            sc = stat_of(0, nullptr);
        } else if (method == 2) {
            sc = stat_of(1, nullptr);
            for (double& m : sc) m = std::sqrt(m);
        } else if (method == 3) {
            mu = stat_of(2, nullptr);
            for (double& m : mu) m /= count;
            HTR_CUDA(cudaMemcpyAsync(dmu->p, mu.data(), sizeof(double) * static_cast<size_t>(F), cudaMemcpyHostToDevice,
                                     c.s));
            sc = stat_of(3, dmu->p);
            for (double& m : sc) m = std::sqrt(m / count);
        }
        for (int f = 0; f < F; ++f)
            if (sc[static_cast<size_t>(f)] == 0.0) {
                sc[static_cast<size_t>(f)] = 1.0;
                fl[static_cast<size_t>(f)] = 1;
            }
        if (scale) std::memcpy(scale, sc.data(), sizeof(double) * static_cast<size_t>(F));
        if (offset) std::memcpy(offset, mu.data(), sizeof(double) * static_cast<size_t>(F));
        if (floored) std::memcpy(floored, fl.data(), sizeof(int32_t) * static_cast<size_t>(F));
        if (!out) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null output pointer");
        HTR_CUDA(cudaMemcpyAsync(dsc->p, sc.data(), sizeof(double) * static_cast<size_t>(F), cudaMemcpyHostToDevice, c.s));
        HTR_CUDA(cudaMemcpyAsync(dmu->p, mu.data(), sizeof(double) * static_cast<size_t>(F), cudaMemcpyHostToDevice, c.s));
        if (out_on_device) {
            if (method == 0) {
                if (out != yt.data())
                    HTR_CUDA(cudaMemcpyAsync(out, yt.data(), sizeof(double) * static_cast<size_t>(n),
                                             cudaMemcpyDeviceToDevice, c.s));
            } else {
                htr::launch_field_apply(yt.data(), n, inner, F, method == 3 ? dmu->p : nullptr, dsc->p, false, out,
                                        c.num_sms, c.s, &c.launches);
            }
            HTR_CUDA(cudaGetLastError());
            HTR_CUDA(cudaStreamSynchronize(c.s));
            return;
        }
        DT o = c.tensor(s);
        if (method == 0)
            HTR_CUDA(cudaMemcpyAsync(o.data(), yt.data(), sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice,
                                     c.s));
        else
            htr::launch_field_apply(yt.data(), n, inner, F, method == 3 ? dmu->p : nullptr, dsc->p, false, o.data(),
                                    c.num_sms, c.s, &c.launches);
        HTR_CUDA(cudaGetLastError());
        output(c, o.data(), n, out, false);
    });
}

htr_status htr_denormalize(htr_context* ctx, const double* y, int32_t y_on_device, const int64_t* shape, int32_t order,
                           int32_t method, int32_t field_axis, const double* scale, const double* offset, double* out,
                           int32_t out_on_device) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        Shape s = to_shape(shape, order);
        if (method < 0 || method > 3) htr::raise(HTR_ERR_INVALID_ARGUMENT, "unknown normalization method");
        const auto [inner, F] = field_view(s, field_axis, order);
        const int64_t n = htrise::shape_product(s);
        DT yt = input(c, y, y_on_device != 0, s);
        if (!out || !scale) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null pointer");
        BufPtr dsc = c.alloc(F), dmu = c.alloc(F);
        HTR_CUDA(cudaMemcpyAsync(dsc->p, scale, sizeof(double) * static_cast<size_t>(F), cudaMemcpyHostToDevice, c.s));
        if (method == 3) {
            if (!offset) htr::raise(HTR_ERR_INVALID_ARGUMENT, "null offset");
            HTR_CUDA(cudaMemcpyAsync(dmu->p, offset, sizeof(double) * static_cast<size_t>(F), cudaMemcpyHostToDevice, c.s));
        }
        DT o;
        double* dst = out;
        if (!out_on_device) {
            o = c.tensor(s);
            dst = o.data();
        }
        if (method == 0) {
            if (dst != yt.data())
                HTR_CUDA(cudaMemcpyAsync(dst, yt.data(), sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice,
                                         c.s));
        } else {
            htr::launch_field_apply(yt.data(), n, inner, F, method == 3 ? dmu->p : nullptr, dsc->p, true, dst, c.num_sms,
                                    c.s, &c.launches);
        }
        HTR_CUDA(cudaGetLastError());
        if (!out_on_device) output(c, dst, n, out, false);
        else HTR_CUDA(cudaStreamSynchronize(c.s));
    });
}

htr_status htr_compute_residual(htr_context* ctx, const double* u, int64_t rows, int64_t r, const double* cm,
                                int64_t cols, double* out) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        DT ut = input(c, u, false, {rows, r});
        DT ct = input(c, cm, false, {rows, cols});
        DT coeff = htr::mode_mul(c, ct, 0, ut.data(), r, rows, 1);  // U^T C
        DT res = c.tensor({rows, cols});
        HTR_CUDA(cudaMemcpyAsync(res.data(), ct.data(), sizeof(double) * static_cast<size_t>(rows * cols),
                                 cudaMemcpyDeviceToDevice, c.s));
        htr::GemmDesc d;  // res -= U coeff
        d.M = rows; d.N1 = cols; d.K1 = r;
        d.A = ut.data(); d.sam = 1; d.sak1 = rows;
        d.B = coeff.data(); d.sbk1 = 1; d.sbn1 = r;
        d.C = res.data(); d.scm = 1; d.scn1 = rows;
        d.alpha = -1.0; d.beta = 1.0;
        htr::run_gemm(c, d);
        output(c, res.data(), rows * cols, out, false);
    });
}

htr_status htr_frobenius_norm(htr_context* ctx, const double* t, int32_t t_on_device, int64_t n, double* out) {
    return guarded(ctx, [&] {
        htr::Context& c = C(ctx);
        DT tt = input(c, t, t_on_device != 0, {n});
        double s = 0.0;
        htr::norm_sq(c, tt.data(), n, &s, nullptr, false);
        *out = std::sqrt(s);
    });
}

}  // extern "C"
