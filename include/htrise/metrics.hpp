// htrise-b200 drop-in: compression metrics and the per-field normalisation
// ledger (reference /root/reference/proj/include/htrise/metrics.hpp:
// NormalizationMethod 15-33, NormalizationParams 38-46, normalize 93-171,
// denormalize 174-197, compression_ratio 200-207, reduction_ratio 210-214,
// relative_test_error 218-237). normalize / denormalize keep the
// reference's host semantics (sequential sums in storage order, so recorded
// ledgers match the reference's bit for bit); normalize_on_device is the
// device prepass the CLI's ingest uses (the batch stays in HBM for the
// compression calls).
#pragma once

#include <algorithm>
#include <cmath>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "htrise/bht.hpp"

namespace htrise {

enum class NormalizationMethod { None, MaxAbs, UnitVec, ZScore };

inline std::string to_string(NormalizationMethod m) {
    switch (m) {
        case NormalizationMethod::MaxAbs: return "maxabs";
        case NormalizationMethod::UnitVec: return "unitvec";
        case NormalizationMethod::ZScore: return "zscore";
        case NormalizationMethod::None: break;
    }
    return "none";
}

inline NormalizationMethod normalization_from_string(const std::string& s) {
    static const std::pair<const char*, NormalizationMethod> names[] = {
        {"none", NormalizationMethod::None},
        {"maxabs", NormalizationMethod::MaxAbs},
        {"unitvec", NormalizationMethod::UnitVec},
        {"zscore", NormalizationMethod::ZScore}};
    for (const auto& [n, m] : names)
        if (s == n) return m;
    throw std::invalid_argument("unknown normalization method: " + s);
}

/// Per-field scalars that undo a normalisation (one entry without a field
/// axis, else one per slice along it); zero scales are floored to 1.
struct NormalizationParams {
    NormalizationMethod method = NormalizationMethod::None;
    std::optional<Index> field_axis;
    std::vector<double> scale;
    std::vector<double> offset;
    std::vector<bool> floored;

    bool operator==(const NormalizationParams&) const = default;
};

namespace detail {

/// Calls fn(field, run pointer, run length) over the contiguous runs of t in
/// storage order (outer index slowest): the reference's accumulation order,
/// which keeps the recorded parameters bit-identical.
template <typename T, typename Fn>
void field_runs(T* data, const Shape& shape, std::optional<Index> axis, Fn&& fn) {
    const Index total = shape_product(shape);
    if (!axis) {
        fn(Index{0}, data, total);
        return;
    }
    require_mode(static_cast<Index>(shape.size()), *axis, "normalize");
    const ModeSplit sp = split_at(shape, *axis);
    for (Index o = 0; o < sp.outer; ++o)
        for (Index f = 0; f < sp.extent; ++f) fn(f, data + sp.inner * (f + sp.extent * o), sp.inner);
}

}  // namespace detail

/// Scale (z-score: also centre) y, per field slice along `field_axis` when
/// given; population standard deviation for z-score.
inline std::pair<DenseTensor, NormalizationParams> normalize(const DenseTensor& y, NormalizationMethod method,
                                                             std::optional<Index> field_axis = std::nullopt) {
    NormalizationParams p;
    p.method = method;
    p.field_axis = field_axis;
    if (field_axis) detail::require_mode(y.order(), *field_axis, "normalize");
    const std::size_t fields = field_axis ? static_cast<std::size_t>(y.extent(*field_axis)) : 1;
    p.scale.assign(fields, method == NormalizationMethod::None ? 1.0 : 0.0);
    p.offset.assign(fields, 0.0);
    p.floored.assign(fields, false);
    if (method == NormalizationMethod::None) return {y, p};

    auto at = [](std::vector<double>& v, Index f) -> double& { return v[static_cast<std::size_t>(f)]; };
    if (method == NormalizationMethod::MaxAbs) {
        detail::field_runs(y.data(), y.shape(), field_axis, [&](Index f, const double* v, Index n) {
            double& m = at(p.scale, f);
            for (Index i = 0; i < n; ++i) m = std::max(m, std::abs(v[i]));
        });
    } else if (method == NormalizationMethod::UnitVec) {
        detail::field_runs(y.data(), y.shape(), field_axis, [&](Index f, const double* v, Index n) {
            double& m = at(p.scale, f);
            for (Index i = 0; i < n; ++i) m += v[i] * v[i];
        });
        for (double& m : p.scale) m = std::sqrt(m);
    } else {
        std::vector<Index> count(fields, 0);
        detail::field_runs(y.data(), y.shape(), field_axis, [&](Index f, const double* v, Index n) {
            double& mu = at(p.offset, f);
            for (Index i = 0; i < n; ++i) mu += v[i];
            count[static_cast<std::size_t>(f)] += n;
        });
        for (std::size_t f = 0; f < fields; ++f) p.offset[f] /= static_cast<double>(count[f]);
        detail::field_runs(y.data(), y.shape(), field_axis, [&](Index f, const double* v, Index n) {
            double& ss = at(p.scale, f);
            const double mu = at(p.offset, f);
            for (Index i = 0; i < n; ++i) ss += (v[i] - mu) * (v[i] - mu);
        });
        for (std::size_t f = 0; f < fields; ++f) p.scale[f] = std::sqrt(p.scale[f] / static_cast<double>(count[f]));
    }
    for (std::size_t f = 0; f < fields; ++f)
        if (p.scale[f] == 0.0) {
            p.scale[f] = 1.0;
            p.floored[f] = true;
        }
    DenseTensor out = y;
    const bool centre = method == NormalizationMethod::ZScore;
    detail::field_runs(out.data(), out.shape(), field_axis, [&](Index f, double* v, Index n) {
        const double mu = centre ? at(p.offset, f) : 0.0, sc = at(p.scale, f);
        for (Index i = 0; i < n; ++i) v[i] = (v[i] - mu) / sc;
    });
    return {std::move(out), std::move(p)};
}

/// normalize on the device (htr_normalize): the batch is uploaded once and
/// stays there, scaled in place, for the compression calls that follow (the
/// CLI's ingest path). Maxima are exact; the unitvec / z-score sums are
/// deterministic tree reductions, so a recorded scale can differ from the
/// host version's sequential sum in the last bit.
inline std::pair<device::DeviceBatch, NormalizationParams> normalize_on_device(
    const DenseTensor& y, NormalizationMethod method, std::optional<Index> field_axis = std::nullopt) {
    NormalizationParams p;
    p.method = method;
    p.field_axis = field_axis;
    if (field_axis) detail::require_mode(y.order(), *field_axis, "normalize");
    const std::size_t fields = field_axis ? static_cast<std::size_t>(y.extent(*field_axis)) : 1;
    p.scale.assign(fields, 1.0);
    p.offset.assign(fields, 0.0);
    std::vector<int32_t> fl(fields, 0);
    device::DeviceBatch b = device::DeviceBatch::upload(y);
    const int32_t m = method == NormalizationMethod::MaxAbs    ? 1
                      : method == NormalizationMethod::UnitVec ? 2
                      : method == NormalizationMethod::ZScore  ? 3
                                                               : 0;
    device::check(htr_normalize(device::ctx(), b.data(), 1, b.shape().data(), static_cast<int32_t>(b.order()), m,
                                field_axis ? static_cast<int32_t>(*field_axis) : -1, b.data(), 1, p.scale.data(),
                                p.offset.data(), fl.data()));
    p.floored.assign(fields, false);
    for (std::size_t f = 0; f < fields; ++f) p.floored[f] = fl[f] != 0;
    return {std::move(b), std::move(p)};
}

/// ||y|| of a device batch (htr_frobenius_norm).
inline double frobenius_norm(const device::DeviceBatch& y) {
    double out = 0.0;
    device::check(htr_frobenius_norm(device::ctx(), y.data(), 1, y.size(), &out));
    return out;
}

/// Inverse of normalize for recorded parameters.
inline DenseTensor denormalize(const DenseTensor& y, const NormalizationParams& p) {
    const std::size_t fields = p.field_axis ? static_cast<std::size_t>(y.extent(*p.field_axis)) : 1;
    if (fields != p.scale.size()) throw std::invalid_argument("denormalize: parameter count mismatch");
    if (p.method == NormalizationMethod::None) return y;
    DenseTensor out = y;
    const bool centre = p.method == NormalizationMethod::ZScore;
    detail::field_runs(out.data(), out.shape(), p.field_axis, [&](Index f, double* v, Index n) {
        const std::size_t fi = static_cast<std::size_t>(f);
        const double mu = centre ? p.offset[fi] : 0.0, sc = p.scale[fi];
        for (Index i = 0; i < n; ++i) v[i] = v[i] * sc + mu;
    });
    return out;
}

inline double compression_ratio(const HTRepresentation& h) {
    if (h.accumulated < 1) throw std::invalid_argument("compression_ratio: empty accumulation");
    return static_cast<double>(shape_product(h.dims)) * static_cast<double>(h.accumulated) /
           static_cast<double>(h.stored_elements());
}

inline double reduction_ratio(const HTRepresentation& h) {
    const DenseTensor& r = h.root();
    return static_cast<double>(shape_product(h.dims)) / static_cast<double>(r.extent(0) * r.extent(1));
}

/// Mean per-tensor relative reconstruction error. Each summand is
/// ||y - decode(encode(y))|| / ||y|| computed on the GPU (htr_relative_error):
/// the reconstruction is compared in HBM and, where the fused decode kernel
/// applies, never materialised.
inline double relative_test_error(const HTRepresentation& h, const std::vector<DenseTensor>& test_set) {
    if (test_set.empty()) throw std::invalid_argument("relative_test_error: empty test set");
    double sum = 0.0;
    for (const DenseTensor& t : test_set) {
        double rel = 0.0;
        device::check(htr_relative_error(device::ctx(), h.device_handle(), t.data(), 0, t.shape().data(),
                                         static_cast<int32_t>(t.order()), &rel));
        sum += rel;
    }
    return sum / static_cast<double>(test_set.size());
}

}  // namespace htrise
