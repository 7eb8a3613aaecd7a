// htrise-b200 drop-in: the bridge from the header API to libhtrise_cuda.so.
//
// Every compute entry point of the reference headers (truncated_svd,
// bht_l2r, encode, decode, reconstruct_slice, ht_rise_update,
// compute_residual, ...) lands here and crosses the C-ABI of
// include/htrise_cuda.h; status codes come back as the reference's exception
// types (std::invalid_argument / std::out_of_range / std::runtime_error).
// Link with -lhtrise_cuda. There is no CPU fallback: without a CUDA device
// every call throws std::runtime_error.
#pragma once

#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "htrise/context.hpp"
#include "htrise/dimension_tree.hpp"
#include "htrise/tensor.hpp"
#include "htrise_cuda.h"

namespace htrise {
namespace device {

/// A batch resident in device memory (htr_device_alloc), canonical layout:
/// what the device-side ingest (normalize_on_device, metrics.hpp) produces and
/// what bht_l2r / encode / ht_rise_update accept without a host copy.
class DeviceBatch {
public:
    DeviceBatch() = default;
    explicit DeviceBatch(Shape shape) : shape_(std::move(shape)) {
        double* p = nullptr;
        check(htr_device_alloc(ctx(), shape_product(shape_), &p));
        p_ = std::shared_ptr<double>(p, [](double* q) { htr_device_free(Context::instance().get(), q); });
    }
    static DeviceBatch upload(const DenseTensor& t) {
        DeviceBatch b(t.shape());
        check(htr_copy(ctx(), b.data(), 1, t.data(), 0, t.size()));
        return b;
    }
    DenseTensor download() const {
        DenseTensor t(shape_);
        check(htr_copy(ctx(), t.data(), 0, data(), 1, size()));
        return t;
    }
    const Shape& shape() const { return shape_; }
    Index order() const { return static_cast<Index>(shape_.size()); }
    Index extent(Index k) const { return shape_.at(static_cast<std::size_t>(k)); }
    Index size() const { return shape_product(shape_); }
    const double* data() const { return p_.get(); }
    double* data() { return p_.get(); }

private:
    Shape shape_;
    std::shared_ptr<double> p_;
};

/// Owning handle of a device-resident representation value.
using RepHandle = std::shared_ptr<htr_rep>;
inline RepHandle wrap(htr_rep* r) {
    return RepHandle(r, [](htr_rep* p) { htr_rep_free(p); });
}

inline std::vector<htr_node> nodes_of(const DimensionTree& t) {
    std::vector<htr_node> out;
    for (Index l = 0; l <= t.depth(); ++l)
        for (const TreeNode& n : t.layer(l)) {
            htr_node h{};
            h.layer = static_cast<int32_t>(n.id.layer);
            h.pos = static_cast<int32_t>(n.id.pos);
            h.kind = n.kind == NodeKind::Root ? HTR_KIND_ROOT : n.kind == NodeKind::Transfer ? HTR_KIND_TRANSFER : HTR_KIND_LEAF;
            h.leaf_dim = static_cast<int32_t>(n.leaf_dim);
            h.succ0 = n.successors.empty() ? -1 : static_cast<int32_t>(n.successors[0].pos);
            h.succ1 = n.successors.empty() ? -1 : static_cast<int32_t>(n.successors[1].pos);
            out.push_back(h);
        }
    return out;
}

inline Shape core_shape(const htr_rep* r, NodeId id) {
    int64_t s[3] = {0, 0, 0};
    int32_t order = 0;
    check(htr_rep_core_shape(r, static_cast<int32_t>(id.layer), static_cast<int32_t>(id.pos), s, &order));
    return Shape(s, s + order);
}

inline DenseTensor fetch_core(const htr_rep* r, NodeId id) {
    Shape s = core_shape(r, id);
    if (shape_product(s) == 0) {
        // an empty root (no slice yet) is not representable as a DenseTensor
        throw std::runtime_error("fetch_core: empty core at " + to_string(id));
    }
    DenseTensor t(s);
    check(htr_rep_core_get(ctx(), r, static_cast<int32_t>(id.layer), static_cast<int32_t>(id.pos), t.data(), 0));
    return t;
}

}  // namespace device
}  // namespace htrise
