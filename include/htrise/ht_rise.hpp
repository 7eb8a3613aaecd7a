// htrise-b200 drop-in: incremental HT-RISE update (reference
// /root/reference/proj/include/htrise/ht_rise.hpp: UpdateOptions 14-17,
// UpdateReport 20-27, compute_residual 31-48, expand_core 53-79,
// pad_with_zeros 83-92, ht_rise_update 99-186).
//
// ht_rise_update runs entirely on the device (libhtrise_cuda.so): the skip
// branch is one fused pass over the batch plus an O(batch) root append that
// shares the input value's cores and root storage (the input stays valid).
#pragma once

#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "htrise/bht.hpp"
#include "htrise/device.hpp"

namespace htrise {

struct UpdateOptions {
    std::optional<double> epsilon_rel;  ///< default: the representation's own
    bool adaptive_budget = false;
};

struct UpdateReport {
    bool skipped = false;
    double proj_error = 0.0;
    double eps_des = 0.0;
    std::map<NodeId, Index> added_ranks;
    RankMap new_ranks;
    double seconds = 0.0;
};

inline Matrix compute_residual(const Matrix& basis, const Matrix& c_unfolded) {
    if (basis.rows() != c_unfolded.rows())
        throw std::invalid_argument("compute_residual: basis has " + std::to_string(basis.rows()) +
                                    " rows, unfolding has " + std::to_string(c_unfolded.rows()));
    Matrix out(c_unfolded.rows(), c_unfolded.cols());
    device::check(htr_compute_residual(device::ctx(), basis.data(), basis.rows(), basis.cols(), c_unfolded.data(),
                                       c_unfolded.cols(), out.data()));
    return out;
}

inline Matrix compute_residual(const HTRepresentation& h, NodeId id, const Matrix& c_unfolded) {
    if (h.tree.node(id).kind == NodeKind::Root) throw std::invalid_argument("compute_residual: root has no basis");
    return compute_residual(h.basis_matrix(id), c_unfolded);
}

/// Append orthonormal directions to a leaf or transfer core (host value op).
inline DenseTensor expand_core(NodeKind kind, const DenseTensor& core, const Matrix& u_new, double orth_tol = 1e-8) {
    if (u_new.cols() == 0) return core;
    if (kind == NodeKind::Root) throw std::invalid_argument("expand_core: root is not a basis core");
    const Shape& s = core.shape();
    const Index alpha = kind == NodeKind::Leaf ? s[0] : s[0] * s[1];
    const Index r_old = kind == NodeKind::Leaf ? s[1] : s[2];
    if (u_new.rows() != alpha)
        throw std::invalid_argument("expand_core: new basis has " + std::to_string(u_new.rows()) + " rows, expected " +
                                    std::to_string(alpha));
    const Matrix u_old = Matrix::from_buffer(core.data(), alpha, r_old);
    const double defect = (u_old.transpose() * u_new).norm();
    if (defect > orth_tol * std::max(1.0, u_new.norm()))
        throw std::invalid_argument("expand_core: new directions not orthogonal to existing basis (defect " +
                                    std::to_string(defect) + ")");
    Matrix joined(alpha, r_old + u_new.cols());
    std::copy(u_old.data(), u_old.data() + u_old.size(), joined.data());
    std::copy(u_new.data(), u_new.data() + u_new.size(), joined.data() + u_old.size());
    if (kind == NodeKind::Leaf) return DenseTensor::from_matrix(joined);
    return reshape(DenseTensor::from_matrix(joined), {s[0], s[1], r_old + u_new.cols()});
}

inline DenseTensor pad_with_zeros(const DenseTensor& core, Index slot, Index r_extra) {
    if (core.order() != 3) throw std::invalid_argument("pad_with_zeros: core must be 3-way");
    if (slot != 0 && slot != 1) throw std::invalid_argument("pad_with_zeros: successor slot must be 0 or 1");
    return pad_zeros(core, slot, r_extra);
}

namespace detail {
inline std::pair<HTRepresentation, UpdateReport> ht_rise_update_at(const HTRepresentation& h, const double* y,
                                                                   int32_t on_device, const Shape& shape,
                                                                   const UpdateOptions& opts) {
    htr_rep* out = nullptr;
    htr_update_report rep{};
    device::check(htr_ht_rise_update(device::ctx(), h.device_handle(), y, on_device, shape.data(),
                                     static_cast<int32_t>(shape.size()), opts.epsilon_rel.value_or(-1.0),
                                     opts.adaptive_budget ? 1 : 0, &out, &rep));
    UpdateReport r;
    r.skipped = rep.skipped != 0;
    r.proj_error = rep.proj_error;
    r.eps_des = rep.eps_des;
    r.seconds = rep.seconds;
    for (int i = 0; i < rep.n_nodes; ++i) {
        const NodeId id{rep.node_layer[i], rep.node_pos[i]};
        r.added_ranks[id] = rep.added_ranks[i];
        r.new_ranks[id] = rep.new_ranks[i];
    }
    return {HTRepresentation::from_device(device::wrap(out)), std::move(r)};
}
}  // namespace detail

inline std::pair<HTRepresentation, UpdateReport> ht_rise_update(const HTRepresentation& h, const DenseTensor& y,
                                                                const UpdateOptions& opts = {}) {
    return detail::ht_rise_update_at(h, y.data(), 0, y.shape(), opts);
}

/// The same on a batch already in device memory (extension: no host copy).
inline std::pair<HTRepresentation, UpdateReport> ht_rise_update(const HTRepresentation& h,
                                                                const device::DeviceBatch& y,
                                                                const UpdateOptions& opts = {}) {
    return detail::ht_rise_update_at(h, y.data(), 1, y.shape(), opts);
}

/// Extension (not in the reference): ht_rise_update over a sequence of
/// batches, each applied to the previous result, as the reference's CLI loop
/// does (tools/main.cpp:225-243). Results are identical to the loop; the
/// library queues batch i+1's skip-path encode before batch i's decision is
/// read back. Returns the value and report after each batch.
inline std::vector<std::pair<HTRepresentation, UpdateReport>> ht_rise_update_many(
    const HTRepresentation& h, const std::vector<DenseTensor>& ys, const UpdateOptions& opts = {}) {
    std::vector<std::pair<HTRepresentation, UpdateReport>> res;
    if (ys.empty()) return res;
    const int32_t order = static_cast<int32_t>(ys.front().order());
    std::vector<const double*> ptrs;
    std::vector<int64_t> shapes;
    for (const DenseTensor& y : ys) {
        if (static_cast<int32_t>(y.order()) != order)
            throw std::invalid_argument("ht_rise_update_many: batches of different tensor order");
        ptrs.push_back(y.data());
        shapes.insert(shapes.end(), y.shape().begin(), y.shape().end());
    }
    std::vector<htr_rep*> outs(ys.size(), nullptr);
    std::vector<htr_update_report> reps(ys.size());
    device::check(htr_ht_rise_update_many(device::ctx(), h.device_handle(), static_cast<int64_t>(ys.size()),
                                          ptrs.data(), 0, shapes.data(), order, opts.epsilon_rel.value_or(-1.0),
                                          opts.adaptive_budget ? 1 : 0, outs.data(), reps.data()));
    for (size_t i = 0; i < ys.size(); ++i) {
        const htr_update_report& rep = reps[i];
        UpdateReport r;
        r.skipped = rep.skipped != 0;
        r.proj_error = rep.proj_error;
        r.eps_des = rep.eps_des;
        r.seconds = rep.seconds;
        for (int k = 0; k < rep.n_nodes; ++k) {
            const NodeId id{rep.node_layer[k], rep.node_pos[k]};
            r.added_ranks[id] = rep.added_ranks[k];
            r.new_ranks[id] = rep.new_ranks[k];
        }
        res.emplace_back(HTRepresentation::from_device(device::wrap(outs[i])), std::move(r));
    }
    return res;
}

}  // namespace htrise
