// htrise-b200 drop-in: error-truncated SVD (reference
// /root/reference/proj/include/htrise/truncated_svd.hpp: TruncatedBasis 17-22,
// truncated_svd 53-100, hosvd_layer 105-123).
//
// The truncation runs on the GPU: Gram of the matrix + one-CTA Jacobi
// eigensolver + the reference's tail-energy rank rule (with a second Gram
// pass re-measuring the small singular values when the tolerance sits near
// the machine floor); see DESIGN.md "K4".
#pragma once

#include <algorithm>
#include <stdexcept>
#include <vector>

#include "htrise/device.hpp"
#include "htrise/tensor.hpp"

namespace htrise {

struct TruncatedBasis {
    Matrix u;                     ///< orthonormal columns, rows x rank
    Index rank = 0;
    double discarded_norm = 0.0;  ///< Frobenius norm of the dropped part
    Vector singular_values;       ///< retained, descending
};

inline TruncatedBasis truncated_svd(const Matrix& m, double eps_abs, Index min_rank = 1) {
    if (m.size() == 0) throw std::invalid_argument("truncated_svd: empty matrix");
    if (!m.allFinite()) throw std::invalid_argument("truncated_svd: non-finite entries");
    if (eps_abs < 0) throw std::invalid_argument("truncated_svd: negative tolerance");
    const Index k = std::min(m.rows(), m.cols());
    std::vector<double> u(static_cast<std::size_t>(m.rows() * std::max<Index>(k, min_rank) + m.rows()));
    std::vector<double> sigma(static_cast<std::size_t>(std::max<Index>(k, 1) + 1));
    int64_t rank = 0;
    double disc = 0.0;
    device::check(htr_truncated_svd(device::ctx(), m.data(), 0, m.rows(), m.cols(), eps_abs, min_rank, u.data(),
                                    sigma.data(), &rank, &disc));
    TruncatedBasis b;
    b.rank = rank;
    b.discarded_norm = disc;
    b.u = Matrix::from_buffer(u.data(), m.rows(), rank);
    b.singular_values = Vector(std::vector<double>(sigma.begin(), sigma.begin() + rank));
    return b;
}

inline std::vector<TruncatedBasis> hosvd_layer(const DenseTensor& c, const std::vector<Index>& modes, double eps_nw,
                                               Index min_rank = 1) {
    std::vector<char> seen(static_cast<std::size_t>(c.order()), 0);
    for (Index m : modes) {
        detail::require_mode(c.order(), m, "hosvd_layer");
        if (seen[static_cast<std::size_t>(m)]) throw std::invalid_argument("hosvd_layer: duplicate mode");
        seen[static_cast<std::size_t>(m)] = 1;
    }
    std::vector<TruncatedBasis> out;
    out.reserve(modes.size());
    for (Index m : modes) out.push_back(truncated_svd(unfold(c, m), eps_nw, min_rank));
    return out;
}

}  // namespace htrise
