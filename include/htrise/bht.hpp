// htrise-b200 drop-in: batch hierarchical Tucker values, BHT-l2r, encode,
// decode (reference /root/reference/proj/include/htrise/bht.hpp:
// kMachineFloorRel 20, effective_eps_rel 22-27, HTRepresentation 34-151,
// LatentBatch 154-158, NodeRecord 161-165, BuildReport 170-174,
// DecompositionOptions 176-178, BhtResult 180-183, adaptive_budget 227-245,
// bht_l2r 251-350, encode 373-401, decode 406-456, pad_latent 460-468,
// reconstruct_slice 472-479).
//
// An HTRepresentation made by bht_l2r / ht_rise_update carries a handle to
// its device-resident copy (libhtrise_cuda.so); encode / decode / updates
// run there. Its non-root cores are mirrored on the host at creation; the
// root (O(accumulated)) is fetched lazily by root() / core({0,0}). A value
// assembled by hand on the host is uploaded on first use.
#pragma once

#include <algorithm>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "htrise/device.hpp"
#include "htrise/dimension_tree.hpp"
#include "htrise/tensor.hpp"
#include "htrise/truncated_svd.hpp"

namespace htrise {

inline constexpr double kMachineFloorRel = 1e-14;

inline double effective_eps_rel(double eps_rel) {
    if (eps_rel < 0 || eps_rel >= 1.0) throw std::invalid_argument("relative tolerance must lie in [0, 1)");
    return eps_rel > 0 ? eps_rel : kMachineFloorRel;
}

struct HTRepresentation {
    DimensionTree tree;
    Shape dims;
    mutable std::vector<std::vector<DenseTensor>> cores;  ///< [layer][pos]; root at [0][0] (lazy)
    Index accumulated = 0;
    double epsilon_rel = 0.0;

    const DenseTensor& core(NodeId id) const {
        if (id.layer == 0 && id.pos == 0) return root();
        return cores.at(static_cast<std::size_t>(id.layer)).at(static_cast<std::size_t>(id.pos));
    }
    DenseTensor& core(NodeId id) {
        (void)root();  // materialise the root before the device copy is dropped
        dev_.reset();  // a mutable core means the device copy may go stale
        root_loaded_ = true;
        return cores.at(static_cast<std::size_t>(id.layer)).at(static_cast<std::size_t>(id.pos));
    }
    const DenseTensor& root() const {
        if (!root_loaded_ && dev_) {
            cores[0][0] = device::fetch_core(dev_.get(), {0, 0});
            root_loaded_ = true;
        }
        return cores.at(0).at(0);
    }

    Index rank(NodeId id) const {
        switch (tree.node(id).kind) {
            case NodeKind::Leaf: return core(id).extent(1);
            case NodeKind::Transfer: return core(id).extent(2);
            case NodeKind::Root: break;
        }
        throw std::invalid_argument("rank: root has no own rank");
    }
    RankMap ranks() const {
        RankMap r;
        for (Index l = 1; l <= tree.depth(); ++l)
            for (const TreeNode& n : tree.layer(l)) r[n.id] = rank(n.id);
        return r;
    }
    Index max_rank() const {
        Index m = 0;
        for (const auto& kv : ranks()) m = std::max(m, kv.second);
        return m;
    }
    Matrix basis_matrix(NodeId id) const {
        const DenseTensor& c = core(id);
        if (tree.node(id).kind == NodeKind::Leaf) return c.as_matrix();
        const Shape& s = c.shape();
        return Matrix::from_buffer(c.data(), s[0] * s[1], s[2]);
    }
    Index stored_elements() const {
        Index total = 0;
        for (Index l = 0; l <= tree.depth(); ++l)
            for (const TreeNode& n : tree.layer(l)) total += core(n.id).size();
        return total;
    }
    IndexSet index_sets(Index batch) const { return IndexSet::build(tree, dims, ranks(), batch); }
    /// max |U^T U - I| over the bases (bht.hpp:101-114). A validation check
    /// of a value (also of one read from disk by the CLI's inspect, which
    /// needs no device): evaluated on the host, entry by entry.
    double orthonormality_defect() const {
        double worst = 0.0;
        for (Index l = 1; l <= tree.depth(); ++l)
            for (const TreeNode& n : tree.layer(l)) {
                const Matrix u = basis_matrix(n.id);
                for (Index a = 0; a < u.cols(); ++a)
                    for (Index b = 0; b <= a; ++b) {
                        double g = 0.0;
                        for (Index i = 0; i < u.rows(); ++i) g += u(i, a) * u(i, b);
                        worst = std::max(worst, std::abs(g - (a == b ? 1.0 : 0.0)));
                    }
            }
        return worst;
    }
    void validate(double tol = 1e-10) const {
        if (static_cast<Index>(dims.size()) != tree.dims())
            throw std::invalid_argument("HTRepresentation: dims/tree mismatch");
        for (Index l = 0; l <= tree.depth(); ++l)
            for (const TreeNode& n : tree.layer(l))
                if (!core(n.id).all_finite()) throw std::runtime_error("HTRepresentation: non-finite core entries");
        const double defect = orthonormality_defect();
        if (!(defect <= tol))
            throw std::runtime_error("HTRepresentation: orthonormality defect " + std::to_string(defect) +
                                     " exceeds " + std::to_string(tol));
        const DenseTensor& r = root();
        if (r.order() != 3 || r.extent(2) != accumulated)
            throw std::invalid_argument("HTRepresentation: root batch extent " + std::to_string(r.extent(2)) +
                                        " != " + std::to_string(accumulated));
        IndexSet sets = index_sets(accumulated);
        for (Index l = 0; l <= tree.depth(); ++l)
            for (const TreeNode& n : tree.layer(l))
                if (core(n.id).shape() != sets.node_set(n.id))
                    throw std::invalid_argument("HTRepresentation: core shape at " + to_string(n.id) +
                                                " inconsistent with its index set");
    }

    /// Device-resident copy (uploaded from the host cores on first use).
    const htr_rep* device_handle() const {
        if (!dev_) {
            std::vector<htr_node> nodes = device::nodes_of(tree);
            std::vector<const double*> ptrs;
            std::vector<int64_t> shapes;
            for (Index l = 0; l <= tree.depth(); ++l)
                for (const TreeNode& n : tree.layer(l)) {
                    const DenseTensor& c = core(n.id);
                    ptrs.push_back(c.data());
                    const Shape& s = c.shape();
                    shapes.push_back(s[0]);
                    shapes.push_back(s[1]);
                    shapes.push_back(s.size() > 2 ? s[2] : 1);
                }
            htr_rep* r = nullptr;
            device::check(htr_rep_import(device::ctx(), nodes.data(), static_cast<int64_t>(nodes.size()), dims.data(),
                                         static_cast<int32_t>(dims.size()), ptrs.data(), shapes.data(), accumulated,
                                         epsilon_rel, &r));
            dev_ = device::wrap(r);
        }
        return dev_.get();
    }

    /// Value built around a device representation: host mirrors of the
    /// non-root cores, root on demand.
    static HTRepresentation from_device(device::RepHandle h) {
        HTRepresentation rep;
        int32_t d = 0;
        int64_t acc = 0, nn = 0;
        double eps = 0.0;
        device::check(htr_rep_info(h.get(), &d, nullptr, nullptr, nullptr, nullptr));
        std::vector<int64_t> dims(static_cast<std::size_t>(std::max<int32_t>(d, 0)));
        device::check(htr_rep_info(h.get(), &d, dims.data(), nullptr, &eps, &nn));
        // the root held here is this rank's shard (the whole stream unsharded)
        device::check(htr_rep_counts(h.get(), &acc, nullptr));
        std::vector<htr_node> nodes(static_cast<std::size_t>(nn));
        device::check(htr_rep_nodes(h.get(), nodes.data(), nn));
        std::vector<std::vector<TreeNode>> layers;
        for (const htr_node& x : nodes) {
            if (static_cast<int32_t>(layers.size()) <= x.layer) layers.resize(static_cast<std::size_t>(x.layer) + 1);
            TreeNode t;
            t.id = {x.layer, x.pos};
            t.kind = x.kind == HTR_KIND_ROOT ? NodeKind::Root : x.kind == HTR_KIND_TRANSFER ? NodeKind::Transfer : NodeKind::Leaf;
            t.leaf_dim = x.leaf_dim;
            if (x.succ0 >= 0) t.successors = {{x.layer + 1, x.succ0}, {x.layer + 1, x.succ1}};
            layers[static_cast<std::size_t>(x.layer)].push_back(t);
        }
        rep.tree = DimensionTree::from_layers(std::move(layers));
        rep.dims = Shape(dims.begin(), dims.end());
        rep.accumulated = acc;
        rep.epsilon_rel = eps;
        rep.cores.resize(static_cast<std::size_t>(rep.tree.depth()) + 1);
        for (Index l = 0; l <= rep.tree.depth(); ++l) {
            rep.cores[static_cast<std::size_t>(l)].resize(static_cast<std::size_t>(rep.tree.layer_size(l)));
            if (l == 0) continue;
            for (const TreeNode& n : rep.tree.layer(l))
                rep.cores[static_cast<std::size_t>(l)][static_cast<std::size_t>(n.id.pos)] = device::fetch_core(h.get(), n.id);
        }
        rep.dev_ = std::move(h);
        rep.root_loaded_ = false;
        return rep;
    }

private:
    mutable device::RepHandle dev_;
    mutable bool root_loaded_ = true;
};

struct LatentBatch {
    DenseTensor slices;  ///< r_{1,1} x r_{1,2} x N
    Index batch_size() const { return slices.extent(2); }
};

struct NodeRecord {
    NodeId id;
    Index rank = 0;
    double discarded_norm = 0.0;
};

struct BuildReport {
    std::vector<NodeRecord> nodes;
    std::vector<double> layer_norms;
    double eps_nw_initial = 0.0;
};

struct DecompositionOptions {
    bool adaptive_budget = false;
};

struct BhtResult {
    HTRepresentation rep;
    BuildReport report;
};

namespace detail {
inline Index svds_below(const DimensionTree& tree, Index l) {
    Index n = 0;
    for (Index k = 1; k < l; ++k) n += tree.layer_size(k);
    return n;
}
}  // namespace detail

inline double adaptive_budget(double eps_abs, double achieved_err_sq, Index svd_remaining) {
    if (svd_remaining < 1) throw std::invalid_argument("adaptive_budget: no SVDs remaining");
    const double budget_sq = eps_abs * eps_abs;
    double rem_sq = budget_sq - achieved_err_sq;
    if (rem_sq < 0) {
        if (achieved_err_sq > budget_sq * (1.0 + 1e-9) + 1e-300)
            throw std::runtime_error("adaptive_budget: error budget exhausted (achieved^2 = " +
                                     std::to_string(achieved_err_sq) + " > eps_abs^2 = " + std::to_string(budget_sq) +
                                     ")");
        rem_sq = 0.0;
    }
    return std::sqrt(rem_sq) / std::sqrt(static_cast<double>(svd_remaining));
}

namespace detail {
inline BhtResult bht_l2r_at(const double* y, int32_t on_device, const Shape& shape, const DimensionTree& tree,
                            double eps_rel, const DecompositionOptions& opts) {
    std::vector<htr_node> nodes = device::nodes_of(tree);
    htr_rep* out = nullptr;
    htr_build_report rep{};
    device::check(htr_bht_l2r(device::ctx(), y, on_device, shape.data(), static_cast<int32_t>(shape.size()),
                              nodes.data(), static_cast<int64_t>(nodes.size()), eps_rel, opts.adaptive_budget ? 1 : 0,
                              &out, &rep));
    BhtResult r{HTRepresentation::from_device(device::wrap(out)), {}};
    for (int i = 0; i < rep.n_records; ++i)
        r.report.nodes.push_back({{rep.rec_layer[i], rep.rec_pos[i]}, rep.rec_rank[i], rep.rec_discarded[i]});
    r.report.layer_norms.assign(rep.layer_norms, rep.layer_norms + rep.n_layer_norms);
    r.report.eps_nw_initial = rep.eps_nw_initial;
    return r;
}
}  // namespace detail

inline BhtResult bht_l2r(const DenseTensor& y, const DimensionTree& tree, double eps_rel,
                         const DecompositionOptions& opts = {}) {
    return detail::bht_l2r_at(y.data(), 0, y.shape(), tree, eps_rel, opts);
}

/// The same on a batch already in device memory (extension: no host copy).
inline BhtResult bht_l2r(const device::DeviceBatch& y, const DimensionTree& tree, double eps_rel,
                         const DecompositionOptions& opts = {}) {
    return detail::bht_l2r_at(y.data(), 1, y.shape(), tree, eps_rel, opts);
}

namespace detail {
inline std::pair<LatentBatch, double> encode_at(const HTRepresentation& h, const double* y, int32_t on_device,
                                                const Shape& shape) {
    const Shape& rs = h.root().shape();  // r11 x r12 x n_acc
    const Index order = static_cast<Index>(shape.size());
    const Index batch = shape.back();
    if (order != h.tree.dims() + 1)
        throw std::invalid_argument("encode: tensor order " + std::to_string(order) + " does not match tree over " +
                                    std::to_string(h.tree.dims()) + " dims plus batch");
    DenseTensor latent({rs[0], rs[1], batch});
    double proj = 0.0;
    device::check(htr_encode(device::ctx(), h.device_handle(), y, on_device, shape.data(), static_cast<int32_t>(order),
                             latent.data(), 0, &proj));
    return {LatentBatch{std::move(latent)}, proj};
}
}  // namespace detail

inline std::pair<LatentBatch, double> encode(const HTRepresentation& h, const DenseTensor& y) {
    return detail::encode_at(h, y.data(), 0, y.shape());
}
inline std::pair<LatentBatch, double> encode(const HTRepresentation& h, const device::DeviceBatch& y) {
    return detail::encode_at(h, y.data(), 1, y.shape());
}

inline DenseTensor decode(const HTRepresentation& h, const LatentBatch& latent) {
    const DenseTensor& l0 = latent.slices;
    Shape out = h.dims;
    out.push_back(l0.order() == 3 ? l0.extent(2) : 1);
    if (l0.order() != 3)
        throw std::invalid_argument("decode: latent ranks " + shape_to_string(l0.shape()) + " do not match root");
    DenseTensor full(out);
    device::check(htr_decode(device::ctx(), h.device_handle(), l0.data(), 0, l0.shape().data(), full.data(), 0));
    return full;
}

inline LatentBatch pad_latent(const LatentBatch& latent, Index r11, Index r12) {
    DenseTensor s = latent.slices;
    if (r11 < s.extent(0) || r12 < s.extent(1)) throw std::invalid_argument("pad_latent: ranks may only grow");
    s = pad_zeros(s, 0, r11 - s.extent(0));
    s = pad_zeros(s, 1, r12 - s.extent(1));
    return {std::move(s)};
}

inline DenseTensor reconstruct_slice(const HTRepresentation& h, Index m) {
    if (m < 1 || m > h.accumulated)
        throw std::out_of_range("reconstruct_slice: index " + std::to_string(m) + " outside 1.." +
                                std::to_string(h.accumulated));
    DenseTensor out(h.dims);
    device::check(htr_reconstruct_slice(device::ctx(), h.device_handle(), m, out.data(), 0));
    return out;
}

}  // namespace htrise
