// htrise-b200 drop-in: dense tensor value type and host tensor algebra.
//
// Mirrors the public surface of the reference header
// /root/reference/proj/include/htrise/tensor.hpp (DenseTensor 42-127,
// unfold/fold 150-205, reshape 209, permute_axes 219, frobenius_norm 269,
// contract 273, mode_multiply 300, ModeFactor/multi_contract 318-380,
// concat/pad_zeros/slice 383-445). The reference builds these on Eigen3,
// which is absent from this image, so this header ships a small
// column-major Matrix/Vector of its own with the subset of the Eigen API the
// htrise interfaces expose (data/rows/cols/operator()/transpose/norm/...).
//
// The arithmetic -- Matrix products, mode_multiply, contract, permute_axes
// and the products multi_contract composes -- runs on the device through
// include/htrise_cuda.h (htr_matmul, htr_mode_multiply, htr_contract,
// htr_permute_axes); what stays on the host is value plumbing (storage,
// unfold/fold/reshape/concat/pad/slice copies, element access).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <initializer_list>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "htrise/context.hpp"

namespace htrise {

using Index = std::int64_t;
using Shape = std::vector<Index>;

inline Index shape_product(const Shape& s) {
    Index p = 1;
    for (Index e : s) p *= e;
    return p;
}

inline std::string shape_to_string(const Shape& s) {
    std::string out = "[";
    for (std::size_t i = 0; i < s.size(); ++i) {
        out += (i ? "x" : "") + std::to_string(s[i]);
    }
    return out + "]";
}

// ---------------------------------------------------------------------------
// Minimal column-major dense linear algebra (stand-in for Eigen::MatrixXd /
// Eigen::VectorXd in the htrise signatures).
// ---------------------------------------------------------------------------

class Vector {
public:
    Vector() = default;
    explicit Vector(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
    Vector(std::initializer_list<double> il) : v_(il) {}
    explicit Vector(std::vector<double> v) : v_(std::move(v)) {}

    static Vector Zero(Index n) { return Vector(n); }
    static Vector Ones(Index n) {
        Vector r(n);
        std::fill(r.v_.begin(), r.v_.end(), 1.0);
        return r;
    }
    static Vector Unit(Index n, Index i) {
        Vector r(n);
        r[i] = 1.0;
        return r;
    }

    Index size() const { return static_cast<Index>(v_.size()); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
    double& operator()(Index i) { return (*this)[i]; }
    double operator()(Index i) const { return (*this)[i]; }

    double squaredNorm() const {
        double s = 0.0;
        for (double x : v_) s += x * x;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    bool allFinite() const {
        for (double x : v_)
            if (!std::isfinite(x)) return false;
        return true;
    }
    Vector head(Index n) const {
        return Vector(std::vector<double>(v_.begin(), v_.begin() + n));
    }
    Vector segment(Index start, Index n) const {
        return Vector(std::vector<double>(v_.begin() + start, v_.begin() + start + n));
    }
    void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }

    Vector operator-(const Vector& o) const { return zip(o, std::minus<double>()); }
    Vector operator+(const Vector& o) const { return zip(o, std::plus<double>()); }
    Vector operator*(double a) const {
        Vector r = *this;
        for (double& x : r.v_) x *= a;
        return r;
    }
    Vector operator/(double a) const { return *this * (1.0 / a); }
    bool operator==(const Vector& o) const { return v_ == o.v_; }
    bool operator!=(const Vector& o) const { return !(*this == o); }

    const std::vector<double>& std_vector() const { return v_; }

private:
    template <typename Op>
    Vector zip(const Vector& o, Op op) const {
        if (o.size() != size()) throw std::invalid_argument("Vector: size mismatch");
        Vector r(size());
        for (std::size_t i = 0; i < v_.size(); ++i) r.v_[i] = op(v_[i], o.v_[i]);
        return r;
    }
    std::vector<double> v_;
};

class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols)
        : rows_(rows), cols_(cols), a_(static_cast<std::size_t>(rows * cols), 0.0) {}

    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    static Matrix Ones(Index r, Index c) {
        Matrix m(r, c);
        std::fill(m.a_.begin(), m.a_.end(), 1.0);
        return m;
    }
    /// Copy of a column-major buffer (Eigen::Map<const Matrix> analogue).
    static Matrix from_buffer(const double* p, Index r, Index c) {
        Matrix m(r, c);
        if (r > 0 && c > 0) std::memcpy(m.a_.data(), p, sizeof(double) * static_cast<std::size_t>(r * c));
        return m;
    }

    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    double& operator()(Index i, Index j) { return a_[static_cast<std::size_t>(i + rows_ * j)]; }
    double operator()(Index i, Index j) const { return a_[static_cast<std::size_t>(i + rows_ * j)]; }

    Matrix transpose() const {
        Matrix t(cols_, rows_);
        for (Index j = 0; j < cols_; ++j)
            for (Index i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
        return t;
    }
    void transposeInPlace() { *this = transpose(); }

    double squaredNorm() const {
        double s = 0.0;
        for (double x : a_) s += x * x;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    bool allFinite() const {
        for (double x : a_)
            if (!std::isfinite(x)) return false;
        return true;
    }
    double maxAbs() const {
        double m = 0.0;
        for (double x : a_) m = std::max(m, std::abs(x));
        return m;
    }
    Matrix leftCols(Index n) const {
        Matrix m(rows_, n);
        if (rows_ > 0 && n > 0) std::memcpy(m.a_.data(), a_.data(), sizeof(double) * static_cast<std::size_t>(rows_ * n));
        return m;
    }
    Matrix col(Index j) const { return block(0, j, rows_, 1); }
    Matrix block(Index r0, Index c0, Index nr, Index nc) const {
        Matrix m(nr, nc);
        for (Index j = 0; j < nc; ++j)
            for (Index i = 0; i < nr; ++i) m(i, j) = (*this)(r0 + i, c0 + j);
        return m;
    }

    /// Product on the device (htr_matmul; Eigen's GEMM in the reference).
    Matrix operator*(const Matrix& b) const {
        if (cols_ != b.rows_) throw std::invalid_argument("Matrix: product shape mismatch");
        Matrix c(rows_, b.cols_);
        if (rows_ == 0 || b.cols_ == 0) return c;
        device::check(htr_matmul(device::ctx(), a_.data(), rows_, cols_, b.a_.data(), b.cols_, c.a_.data()));
        return c;
    }
    Matrix operator-(const Matrix& b) const { return zip(b, std::minus<double>()); }
    Matrix operator+(const Matrix& b) const { return zip(b, std::plus<double>()); }
    Matrix operator*(double s) const {
        Matrix r = *this;
        for (double& x : r.a_) x *= s;
        return r;
    }
    bool operator==(const Matrix& o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ && a_ == o.a_;
    }

private:
    template <typename Op>
    Matrix zip(const Matrix& b, Op op) const {
        if (rows_ != b.rows_ || cols_ != b.cols_)
            throw std::invalid_argument("Matrix: shape mismatch");
        Matrix r(rows_, cols_);
        for (std::size_t i = 0; i < a_.size(); ++i) r.a_[i] = op(a_[i], b.a_[i]);
        return r;
    }
    Index rows_ = 0, cols_ = 0;
    std::vector<double> a_;
};

// ---------------------------------------------------------------------------
// DenseTensor: canonical first-index-fastest f64 buffer (reference
// tensor.hpp:36-41 layout contract).
// ---------------------------------------------------------------------------

class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(Shape shape) : shape_(std::move(shape)) {
        data_ = Vector(validated(shape_));
    }
    DenseTensor(Shape shape, Vector data) : shape_(std::move(shape)), data_(std::move(data)) {
        const Index need = validated(shape_);
        if (data_.size() != need) {
            throw std::invalid_argument("DenseTensor: buffer has " + std::to_string(data_.size()) +
                                        " entries, shape " + shape_to_string(shape_) + " needs " +
                                        std::to_string(need));
        }
    }

    static DenseTensor from_matrix(const Matrix& m) {
        Vector v(m.size());
        if (m.size()) std::memcpy(v.data(), m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
        return DenseTensor({m.rows(), m.cols()}, std::move(v));
    }
    Matrix as_matrix() const {
        if (order() != 2)
            throw std::invalid_argument("as_matrix: tensor has order " + std::to_string(order()));
        return Matrix::from_buffer(data(), shape_[0], shape_[1]);
    }

    const Shape& shape() const { return shape_; }
    Index extent(Index mode) const { return shape_.at(static_cast<std::size_t>(mode)); }
    Index order() const { return static_cast<Index>(shape_.size()); }
    Index size() const { return data_.size(); }
    const Vector& values() const { return data_; }
    Vector& values_mut() { return data_; }
    const double* data() const { return data_.data(); }
    double* data() { return data_.data(); }

    double operator()(const Shape& idx) const { return data_[linear(idx)]; }
    double& operator()(const Shape& idx) { return data_[linear(idx)]; }
    bool all_finite() const { return data_.allFinite(); }
    bool operator==(const DenseTensor& o) const { return shape_ == o.shape_ && data_ == o.data_; }

private:
    static Index validated(const Shape& s) {
        if (s.empty()) throw std::invalid_argument("DenseTensor: empty shape");
        for (Index e : s)
            if (e < 1) throw std::invalid_argument("DenseTensor: extent " + std::to_string(e) + " < 1");
        return shape_product(s);
    }
    Index linear(const Shape& idx) const {
        if (idx.size() != shape_.size())
            throw std::invalid_argument("DenseTensor: index order mismatch");
        Index off = 0;
        for (std::size_t k = shape_.size(); k-- > 0;) {
            if (idx[k] < 0 || idx[k] >= shape_[k])
                throw std::out_of_range("DenseTensor: index out of range");
            off = off * shape_[k] + idx[k];
        }
        return off;
    }
    Shape shape_;
    Vector data_;
};

namespace detail {

inline void require_mode(Index order, Index mode, const char* who) {
    if (mode < 0 || mode >= order) {
        throw std::invalid_argument(std::string(who) + ": mode " + std::to_string(mode) +
                                    " out of range for order " + std::to_string(order));
    }
}

/// (inner, extent, outer) split of a canonical buffer around `mode`.
struct ModeSplit {
    Index inner = 1, extent = 1, outer = 1;
};
inline ModeSplit split_at(const Shape& s, Index mode) {
    ModeSplit m;
    for (Index k = 0; k < mode; ++k) m.inner *= s[static_cast<std::size_t>(k)];
    m.extent = s[static_cast<std::size_t>(mode)];
    for (std::size_t k = static_cast<std::size_t>(mode) + 1; k < s.size(); ++k) m.outer *= s[k];
    return m;
}

}  // namespace detail

/// Mode-k matricization: row = index along `mode`, column = remaining
/// indices enumerated in canonical order (reference tensor.hpp:146-172).
inline Matrix unfold(const DenseTensor& t, Index mode) {
    detail::require_mode(t.order(), mode, "unfold");
    const auto sp = detail::split_at(t.shape(), mode);
    Matrix m(sp.extent, sp.inner * sp.outer);
    const double* src = t.data();
    for (Index o = 0; o < sp.outer; ++o)
        for (Index r = 0; r < sp.extent; ++r)
            for (Index i = 0; i < sp.inner; ++i)
                m(r, i + sp.inner * o) = src[i + sp.inner * (r + sp.extent * o)];
    return m;
}

/// Exact inverse of unfold (reference tensor.hpp:176-205).
inline DenseTensor fold(const Matrix& m, const Shape& shape, Index mode) {
    if (mode < 0 || mode >= static_cast<Index>(shape.size()))
        throw std::invalid_argument("fold: mode out of range");
    const auto sp = detail::split_at(shape, mode);
    if (m.rows() != sp.extent || m.rows() * m.cols() != shape_product(shape)) {
        throw std::invalid_argument("fold: matrix " + std::to_string(m.rows()) + "x" +
                                    std::to_string(m.cols()) + " inconsistent with shape " +
                                    shape_to_string(shape) + " at mode " + std::to_string(mode));
    }
    DenseTensor t(shape);
    double* dst = t.data();
    for (Index o = 0; o < sp.outer; ++o)
        for (Index r = 0; r < sp.extent; ++r)
            for (Index i = 0; i < sp.inner; ++i)
                dst[i + sp.inner * (r + sp.extent * o)] = m(r, i + sp.inner * o);
    return t;
}

inline DenseTensor reshape(const DenseTensor& t, const Shape& index_set) {
    if (shape_product(index_set) != t.size()) {
        throw std::invalid_argument("reshape: product of " + shape_to_string(index_set) +
                                    " != " + std::to_string(t.size()) + " elements");
    }
    return DenseTensor(index_set, t.values());
}

/// Result mode k is input mode perm[k] (reference tensor.hpp:219-267).
inline DenseTensor permute_axes(const DenseTensor& t, const std::vector<Index>& perm) {
    const Index d = t.order();
    if (static_cast<Index>(perm.size()) != d)
        throw std::invalid_argument("permute_axes: permutation order mismatch");
    std::vector<char> used(static_cast<std::size_t>(d), 0);
    for (Index p : perm) {
        if (p < 0 || p >= d || used[static_cast<std::size_t>(p)])
            throw std::invalid_argument("permute_axes: invalid permutation");
        used[static_cast<std::size_t>(p)] = 1;
    }
    Shape out_shape(static_cast<std::size_t>(d));
    for (Index k = 0; k < d; ++k) out_shape[static_cast<std::size_t>(k)] = t.extent(perm[static_cast<std::size_t>(k)]);
    DenseTensor out(out_shape);
    device::check(htr_permute_axes(device::ctx(), t.data(), t.shape().data(), static_cast<int32_t>(d), perm.data(),
                                   out.data()));
    return out;
}

/// ||t|| on the device (htr_frobenius_norm).
inline double frobenius_norm(const DenseTensor& t) {
    double out = 0.0;
    device::check(htr_frobenius_norm(device::ctx(), t.data(), 0, t.size(), &out));
    return out;
}

/// Contract a(mode da) with b(mode db); result modes: a's rest then b's rest.
inline DenseTensor contract(const DenseTensor& a, Index da, const DenseTensor& b, Index db) {
    detail::require_mode(a.order(), da, "contract");
    detail::require_mode(b.order(), db, "contract");
    if (a.extent(da) != b.extent(db)) {
        throw std::invalid_argument("contract: extent mismatch " + std::to_string(a.extent(da)) +
                                    " vs " + std::to_string(b.extent(db)));
    }
    Shape out;
    for (Index k = 0; k < a.order(); ++k)
        if (k != da) out.push_back(a.extent(k));
    for (Index k = 0; k < b.order(); ++k)
        if (k != db) out.push_back(b.extent(k));
    if (out.empty()) out = {1};
    DenseTensor r(out);
    device::check(htr_contract(device::ctx(), a.data(), a.shape().data(), static_cast<int32_t>(a.order()),
                               static_cast<int32_t>(da), b.data(), b.shape().data(), static_cast<int32_t>(b.order()),
                               static_cast<int32_t>(db), r.data()));
    return r;
}

/// Replace mode `mode` of t by the rows of m (q x extent(mode)).
inline DenseTensor mode_multiply(const DenseTensor& t, Index mode, const Matrix& m) {
    detail::require_mode(t.order(), mode, "mode_multiply");
    if (m.cols() != t.extent(mode)) {
        throw std::invalid_argument("mode_multiply: factor has " + std::to_string(m.cols()) +
                                    " cols, mode extent is " + std::to_string(t.extent(mode)));
    }
    Shape out = t.shape();
    out[static_cast<std::size_t>(mode)] = m.rows();
    DenseTensor r(out);
    if (m.rows() == 0) return r;
    device::check(htr_mode_multiply(device::ctx(), t.data(), 0, t.shape().data(), static_cast<int32_t>(t.order()),
                                    static_cast<int32_t>(mode), m.data(), m.rows(), r.data(), 0));
    return r;
}

/// One factor of a multi-index contraction (reference tensor.hpp:318-323).
struct ModeFactor {
    DenseTensor tensor;
    Index target_mode = 0;
    Index axis = -1;  // -1: last axis
};

inline DenseTensor multi_contract(const DenseTensor& t, std::vector<ModeFactor> factors) {
    std::stable_sort(factors.begin(), factors.end(),
                     [](const ModeFactor& a, const ModeFactor& b) { return a.target_mode < b.target_mode; });
    for (std::size_t i = 1; i < factors.size(); ++i)
        if (factors[i].target_mode == factors[i - 1].target_mode)
            throw std::invalid_argument("multi_contract: duplicate target mode " +
                                        std::to_string(factors[i].target_mode));
    DenseTensor c = t;
    Index inserted = 0;
    for (const ModeFactor& f : factors) {
        const Index mode = f.target_mode + inserted;
        detail::require_mode(c.order(), mode, "multi_contract");
        const Index fo = f.tensor.order();
        const Index axis = f.axis < 0 ? fo - 1 : f.axis;
        if (fo == 2) {
            if (axis != 0 && axis != 1) throw std::invalid_argument("multi_contract: bad 2-way axis");
            Matrix m = f.tensor.as_matrix();
            c = mode_multiply(c, mode, axis == 0 ? m.transpose() : m);
        } else if (fo == 3) {
            if (axis != 2)
                throw std::invalid_argument("multi_contract: 3-way factors contract their last axis");
            const Shape& fs = f.tensor.shape();
            Matrix m = Matrix::from_buffer(f.tensor.data(), fs[0] * fs[1], fs[2]);
            if (m.cols() != c.extent(mode))
                throw std::invalid_argument("multi_contract: extent mismatch at mode " +
                                            std::to_string(f.target_mode));
            DenseTensor merged = mode_multiply(c, mode, m);
            Shape split = c.shape();
            split[static_cast<std::size_t>(mode)] = fs[0];
            split.insert(split.begin() + mode + 1, fs[1]);
            c = reshape(merged, split);
            ++inserted;
        } else {
            throw std::invalid_argument("multi_contract: factors must be 2- or 3-way");
        }
    }
    return c;
}

inline DenseTensor concat(const DenseTensor& a, const DenseTensor& b, Index k) {
    detail::require_mode(a.order(), k, "concat");
    if (a.order() != b.order()) throw std::invalid_argument("concat: order mismatch");
    for (Index m = 0; m < a.order(); ++m)
        if (m != k && a.extent(m) != b.extent(m))
            throw std::invalid_argument("concat: shapes differ off mode " + std::to_string(k) + ": " +
                                        shape_to_string(a.shape()) + " vs " + shape_to_string(b.shape()));
    const auto sa = detail::split_at(a.shape(), k);
    const auto sb = detail::split_at(b.shape(), k);
    Shape out_shape = a.shape();
    out_shape[static_cast<std::size_t>(k)] += b.extent(k);
    DenseTensor out(out_shape);
    const Index la = sa.inner * sa.extent, lb = sb.inner * sb.extent;
    double* dst = out.data();
    for (Index o = 0; o < sa.outer; ++o) {
        std::memcpy(dst, a.data() + la * o, sizeof(double) * static_cast<std::size_t>(la));
        std::memcpy(dst + la, b.data() + lb * o, sizeof(double) * static_cast<std::size_t>(lb));
        dst += la + lb;
    }
    return out;
}

inline DenseTensor pad_zeros(const DenseTensor& t, Index k, Index extra) {
    if (extra == 0) return t;
    if (extra < 0) throw std::invalid_argument("pad_zeros: negative pad");
    detail::require_mode(t.order(), k, "pad_zeros");
    Shape z = t.shape();
    z[static_cast<std::size_t>(k)] = extra;
    return concat(t, DenseTensor(z), k);
}

inline DenseTensor slice(const DenseTensor& t, Index k, Index from, Index count) {
    detail::require_mode(t.order(), k, "slice");
    if (from < 0 || count < 1 || from + count > t.extent(k))
        throw std::out_of_range("slice: range out of bounds");
    const auto sp = detail::split_at(t.shape(), k);
    Shape out_shape = t.shape();
    out_shape[static_cast<std::size_t>(k)] = count;
    DenseTensor out(out_shape);
    const Index run = sp.inner * count;
    for (Index o = 0; o < sp.outer; ++o)
        std::memcpy(out.data() + run * o, t.data() + sp.inner * (from + sp.extent * o),
                    sizeof(double) * static_cast<std::size_t>(run));
    return out;
}

}  // namespace htrise
