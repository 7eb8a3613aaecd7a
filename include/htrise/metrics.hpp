// htrise-b200 drop-in: compression metrics (reference
// /root/reference/proj/include/htrise/metrics.hpp: compression_ratio 200-207,
// reduction_ratio 210-214, relative_test_error 218-237). Per-field
// normalisation (metrics.hpp:93-197) is outside the accelerated path; see
// DESIGN.md "Out of scope".
#pragma once

#include <stdexcept>
#include <vector>

#include "htrise/bht.hpp"

namespace htrise {

inline double compression_ratio(const HTRepresentation& h) {
    if (h.accumulated < 1) throw std::invalid_argument("compression_ratio: empty accumulation");
    return static_cast<double>(shape_product(h.dims)) * static_cast<double>(h.accumulated) /
           static_cast<double>(h.stored_elements());
}

inline double reduction_ratio(const HTRepresentation& h) {
    const DenseTensor& r = h.root();
    return static_cast<double>(shape_product(h.dims)) / static_cast<double>(r.extent(0) * r.extent(1));
}

/// Mean per-tensor relative reconstruction error (encode + decode on the GPU).
inline double relative_test_error(const HTRepresentation& h, const std::vector<DenseTensor>& test_set) {
    if (test_set.empty()) throw std::invalid_argument("relative_test_error: empty test set");
    double sum = 0.0;
    for (const DenseTensor& t : test_set) {
        Shape with_batch = t.shape();
        if (t.order() == h.tree.dims()) with_batch.push_back(1);
        DenseTensor y = reshape(t, with_batch);
        DenseTensor back = decode(h, encode(h, y).first);
        const double ny = frobenius_norm(y);
        if (ny == 0.0) continue;
        sum += (y.values() - back.values()).norm() / ny;
    }
    return sum / static_cast<double>(test_set.size());
}

}  // namespace htrise
