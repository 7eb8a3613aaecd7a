// Drop-in check: reference-style tests written against the htrise C++ API
// (include/htrise/*.hpp), running on the GPU through libhtrise_cuda.so.
// Mirrors cases of /root/reference/proj/tests/test_bht.cpp,
// test_ht_rise.cpp, test_truncated_svd.cpp and test_metrics.cpp with plain
// asserts (Catch2 is not available here).
#include <htrise/htrise.hpp>

#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>

using namespace htrise;

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);       \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static DenseTensor random_tensor(const Shape& shape, std::mt19937_64& rng) {
    std::normal_distribution<double> dist;
    Vector v(shape_product(shape));
    for (Index i = 0; i < v.size(); ++i) v[i] = dist(rng);
    return DenseTensor(shape, std::move(v));
}

static Matrix random_orthonormal(Index rows, Index cols, std::mt19937_64& rng) {
    // Gram-Schmidt (twice) on a Gaussian matrix
    std::normal_distribution<double> dist;
    Matrix q(rows, cols);
    for (Index j = 0; j < cols; ++j) {
        for (Index i = 0; i < rows; ++i) q(i, j) = dist(rng);
        for (int pass = 0; pass < 2; ++pass)
            for (Index k = 0; k < j; ++k) {
                double d = 0;
                for (Index i = 0; i < rows; ++i) d += q(i, k) * q(i, j);
                for (Index i = 0; i < rows; ++i) q(i, j) -= d * q(i, k);
            }
        double n = 0;
        for (Index i = 0; i < rows; ++i) n += q(i, j) * q(i, j);
        n = std::sqrt(n);
        for (Index i = 0; i < rows; ++i) q(i, j) /= n;
    }
    return q;
}

static DenseTensor tucker_family_batch(const std::vector<Matrix>& bases, Index n, std::mt19937_64& rng) {
    Shape core_shape, out_shape;
    for (const Matrix& b : bases) {
        core_shape.push_back(b.cols());
        out_shape.push_back(b.rows());
    }
    Shape batch_shape = out_shape;
    batch_shape.push_back(n);
    DenseTensor out(batch_shape);
    const Index slice = shape_product(out_shape);
    for (Index s = 0; s < n; ++s) {
        DenseTensor t = random_tensor(core_shape, rng);
        for (std::size_t k = 0; k < bases.size(); ++k) t = mode_multiply(t, static_cast<Index>(k), bases[k]);
        std::copy(t.data(), t.data() + slice, out.data() + s * slice);
    }
    return out;
}

static double rel_err(const DenseTensor& a, const DenseTensor& b) {
    return (a.values() - b.values()).norm() / a.values().norm();
}

int main() {
    std::mt19937_64 rng(77002);

    {  // tensor algebra on the device (tensor.hpp:219-380) against plain loops
        DenseTensor a = random_tensor({3, 4, 5}, rng), b = random_tensor({6, 4, 2}, rng);
        DenseTensor c = contract(a, 1, b, 1);  // [3, 5, 6, 2]
        CHECK((c.shape() == Shape{3, 5, 6, 2}));
        double worst = 0.0;
        for (Index i = 0; i < 3; ++i)
            for (Index k = 0; k < 5; ++k)
                for (Index p = 0; p < 6; ++p)
                    for (Index q = 0; q < 2; ++q) {
                        double s = 0.0;
                        for (Index j = 0; j < 4; ++j) s += a({i, j, k}) * b({p, j, q});
                        worst = std::max(worst, std::abs(c({i, k, p, q}) - s));
                    }
        CHECK(worst <= 1e-12);
        CHECK(throws<std::invalid_argument>([&] { contract(a, 0, b, 0); }));
        DenseTensor pt = permute_axes(a, {2, 0, 1});  // out(k, i, j) = a(i, j, k)
        CHECK((pt.shape() == Shape{5, 3, 4}));
        bool same = true;
        for (Index i = 0; i < 3; ++i)
            for (Index j = 0; j < 4; ++j)
                for (Index k = 0; k < 5; ++k) same = same && pt({k, i, j}) == a({i, j, k});
        CHECK(same);
        CHECK(throws<std::invalid_argument>([&] { permute_axes(a, {0, 0, 1}); }));
        Matrix m = random_orthonormal(7, 4, rng), n = random_orthonormal(4, 3, rng);
        Matrix mn = m * n;
        double err = 0.0;
        for (Index i = 0; i < 7; ++i)
            for (Index j = 0; j < 3; ++j) {
                double s = 0.0;
                for (Index k = 0; k < 4; ++k) s += m(i, k) * n(k, j);
                err = std::max(err, std::abs(mn(i, j) - s));
            }
        CHECK(err <= 1e-14);
        CHECK(throws<std::invalid_argument>([&] { (void)(m * m); }));
        DenseTensor mm = mode_multiply(a, 2, random_orthonormal(5, 2, rng).transpose());
        CHECK((mm.shape() == Shape{3, 4, 2}));
    }

    {  // test_truncated_svd.cpp:22-36
        Matrix m = Matrix::Zero(2, 2);
        m(0, 0) = 4.0;
        m(1, 1) = 3.0;
        TruncatedBasis keep1 = truncated_svd(m, 3.0);
        CHECK(keep1.rank == 1);
        CHECK(std::abs(std::abs(keep1.u(0, 0)) - 1.0) <= 1e-12);
        CHECK(std::abs(keep1.discarded_norm - 3.0) <= 1e-12);
        CHECK(truncated_svd(m, 2.9).rank == 2);
        TruncatedBasis z = truncated_svd(Matrix::Zero(3, 3), 0.1);
        CHECK(z.rank == 1 && z.u(0, 0) == 1.0 && z.u(1, 0) == 0.0);
        CHECK(truncated_svd(Matrix::Zero(3, 3), 0.1, 0).rank == 0);
        CHECK(throws<std::invalid_argument>([&] { truncated_svd(Matrix::Ones(2, 2), -1.0); }));
    }
    {  // test_bht.cpp:42-53 rank-1 exactness
        Shape dims = {3, 4, 2, 3};
        Shape shape = dims;
        shape.push_back(5);
        DenseTensor y(shape);
        for (Index flat = 0; flat < y.size(); ++flat) {
            Index rem = flat;
            double v = 1.0;
            for (std::size_t k = 0; k < dims.size(); ++k) {
                const Index i = rem % dims[k];
                rem /= dims[k];
                v *= 1.0 + double(i + 1) / double(k + 2);
            }
            y.data()[flat] = v;
        }
        auto [rep, report] = bht_l2r(y, DimensionTree::balanced(4), 0.3);
        for (const auto& kv : rep.ranks()) CHECK(kv.second == 1);
        rep.validate();
        auto [latent, proj] = encode(rep, y);
        CHECK(rel_err(y, decode(rep, latent)) <= 1e-12);
    }
    {  // test_bht.cpp:55-63 node-wise tolerance KAT
        DenseTensor y = random_tensor({2, 2, 2, 2, 2, 3}, rng);
        DenseTensor unit(y.shape(), y.values() / y.values().norm());
        auto [rep, report] = bht_l2r(unit, DimensionTree::balanced(5), 0.1);
        CHECK(std::abs(report.eps_nw_initial - 0.1 / std::sqrt(8.0)) <= 1e-12);
    }
    {  // test_bht.cpp:266-288 bound + norm identity over orders
        std::uniform_int_distribution<Index> ext(2, 5), nb(1, 6);
        for (Index d : {2, 3, 4, 5, 6}) {
            for (double eps : {0.3, 0.05}) {
                Shape shape;
                for (Index k = 0; k < d; ++k) shape.push_back(ext(rng));
                shape.push_back(nb(rng));
                DenseTensor y = random_tensor(shape, rng);
                auto [rep, report] = bht_l2r(y, DimensionTree::balanced(d), eps);
                rep.validate();
                auto [latent, proj] = encode(rep, y);
                DenseTensor back = decode(rep, latent);
                CHECK(rel_err(y, back) <= eps + 1e-9);
                const double ny2 = y.values().squaredNorm();
                const double nl2 = latent.slices.values().squaredNorm();
                const double diff2 = (y.values() - back.values()).squaredNorm();
                CHECK(std::abs((ny2 - nl2) - diff2) <= 1e-9 * ny2);
            }
        }
    }
    {  // test_bht.cpp:319-339 malformed inputs
        DimensionTree tree = DimensionTree::balanced(3);
        CHECK(throws<std::invalid_argument>([&] { bht_l2r(DenseTensor({2, 2, 2}), tree, 0.1); }));
        Vector bad = Vector::Zero(16);
        bad[3] = std::nan("");
        CHECK(throws<std::invalid_argument>([&] { bht_l2r(DenseTensor({2, 2, 2, 2}, bad), tree, 0.1); }));
        CHECK(throws<std::invalid_argument>([&] { bht_l2r(DenseTensor({2, 2, 2, 2}), tree, 1.5); }));
        DenseTensor y = random_tensor({2, 2, 2, 2}, rng);
        auto [rep, report] = bht_l2r(y, tree, 0.1);
        CHECK(throws<std::invalid_argument>([&] { encode(rep, DenseTensor({2, 3, 2, 2})); }));
        CHECK(throws<std::out_of_range>([&] { reconstruct_slice(rep, 0); }));
        CHECK(throws<std::out_of_range>([&] { reconstruct_slice(rep, 3); }));
    }
    {  // test_ht_rise.cpp:139-163 skip branch keeps non-root cores bit-identical
        std::mt19937_64 r2(90210);
        DenseTensor y = random_tensor({3, 3, 3, 4}, r2);
        auto [rep, report] = bht_l2r(y, DimensionTree::balanced(3), 0.2);
        auto [rep2, update] = ht_rise_update(rep, y);
        CHECK(update.skipped);
        CHECK(update.proj_error <= update.eps_des);
        CHECK(rep2.accumulated == 8 && rep2.root().extent(2) == 8);
        for (const auto& kv : update.added_ranks) CHECK(kv.second == 0);
        for (Index l = 1; l <= rep.tree.depth(); ++l)
            for (const TreeNode& n : rep.tree.layer(l)) CHECK(rep2.core(n.id) == rep.core(n.id));
    }
    {  // test_ht_rise.cpp:165-190 a fixed multilinear family saturates and skips
        std::mt19937_64 r3(4242);
        std::vector<Matrix> bases;
        for (Index k = 0; k < 4; ++k) bases.push_back(random_orthonormal(5, 2, r3));
        auto [first, report] = bht_l2r(tucker_family_batch(bases, 3, r3), DimensionTree::balanced(4), 1e-8);
        HTRepresentation rep = first;
        int skips = 0;
        for (int k = 0; k < 12; ++k) {
            auto [next, update] = ht_rise_update(rep, tucker_family_batch(bases, 3, r3));
            rep = std::move(next);
            if (k >= 2) {
                CHECK(update.skipped);
                skips += update.skipped ? 1 : 0;
            }
        }
        CHECK(skips == 10);
        for (Index l = 1; l <= rep.tree.depth(); ++l)
            for (const TreeNode& n : rep.tree.layer(l))
                if (n.kind == NodeKind::Leaf) CHECK(rep.rank(n.id) == 2);
        rep.validate();
    }
    {  // test_ht_rise.cpp:202-257 past slices immutable + per-batch bound
        std::mt19937_64 r4(262626);
        const double eps = 0.25;
        std::uniform_int_distribution<Index> nb(1, 4);
        std::vector<DenseTensor> batches;
        for (int k = 0; k < 8; ++k) batches.push_back(random_tensor({3, 4, 3, nb(r4)}, r4));
        auto [rep0, report] = bht_l2r(batches[0], DimensionTree::balanced(3), eps);
        HTRepresentation rep = rep0;
        std::vector<DenseTensor> snaps;
        for (Index m = 1; m <= rep.accumulated; ++m) snaps.push_back(reconstruct_slice(rep, m));
        for (std::size_t k = 1; k < batches.size(); ++k) {
            auto [next, update] = ht_rise_update(rep, batches[k]);
            rep = std::move(next);
            rep.validate();
            for (std::size_t m = 0; m < snaps.size(); ++m) {
                DenseTensor again = reconstruct_slice(rep, static_cast<Index>(m) + 1);
                CHECK((again.values() - snaps[m].values()).norm() <= 1e-10 * frobenius_norm(snaps[m]));
            }
            for (Index m = static_cast<Index>(snaps.size()) + 1; m <= rep.accumulated; ++m)
                snaps.push_back(reconstruct_slice(rep, m));
        }
        Index offset = 0;
        for (const DenseTensor& b : batches) {
            const Index n = b.extent(3);
            double err_sq = 0.0;
            const Index slice = b.size() / n;
            for (Index m = 0; m < n; ++m) {
                DenseTensor orig({3, 4, 3}, b.values().segment(m * slice, slice));
                err_sq += (orig.values() - reconstruct_slice(rep, offset + m + 1).values()).squaredNorm();
            }
            CHECK(std::sqrt(err_sq) <= eps * frobenius_norm(b) + 1e-9);
            offset += n;
        }
    }
    {  // extension: ht_rise_update_many == the per-batch loop (random batches
       // expand every step; a (1,(2,3)) family stream skips on the fused path)
        std::mt19937_64 r6(8080);
        std::uniform_int_distribution<Index> nb(1, 4);
        std::vector<DenseTensor> batches;
        for (int k = 0; k < 6; ++k) batches.push_back(random_tensor({3, 4, 3, nb(r6)}, r6));
        auto [rep0, report] = bht_l2r(batches[0], DimensionTree::balanced(3), 0.25);
        std::vector<DenseTensor> rest(batches.begin() + 1, batches.end());
        auto many = ht_rise_update_many(rep0, rest);
        CHECK(many.size() == rest.size());
        HTRepresentation rep = rep0;
        for (std::size_t k = 0; k < rest.size(); ++k) {
            auto [next, update] = ht_rise_update(rep, rest[k]);
            rep = std::move(next);
            CHECK(update.skipped == many[k].second.skipped);
            CHECK(update.proj_error == many[k].second.proj_error);
            CHECK(update.new_ranks == many[k].second.new_ranks);
            CHECK(rep.accumulated == many[k].first.accumulated);
        }
        for (Index m = 1; m <= rep.accumulated; ++m)
            CHECK(reconstruct_slice(rep, m) == reconstruct_slice(many.back().first, m));

        std::vector<Matrix> bases;
        for (Index n : {64, 64, 16}) bases.push_back(random_orthonormal(n, 3, r6));
        DimensionTree t123 = DimensionTree::from_layers(
            {{TreeNode{{0, 0}, NodeKind::Root, {{1, 0}, {1, 1}}}},
             {TreeNode{{1, 0}, NodeKind::Leaf, {}, {0, 0}, 0}, TreeNode{{1, 1}, NodeKind::Transfer, {{2, 0}, {2, 1}}}},
             {TreeNode{{2, 0}, NodeKind::Leaf, {}, {0, 0}, 1}, TreeNode{{2, 1}, NodeKind::Leaf, {}, {0, 0}, 2}}});
        auto [f0, frep] = bht_l2r(tucker_family_batch(bases, 3, r6), t123, 1e-6);
        std::vector<DenseTensor> fam;
        for (int k = 0; k < 5; ++k) fam.push_back(tucker_family_batch(bases, 2, r6));
        auto fm = ht_rise_update_many(f0, fam);
        HTRepresentation fr = f0;
        for (std::size_t k = 0; k < fam.size(); ++k) {
            auto [next, update] = ht_rise_update(fr, fam[k]);
            fr = std::move(next);
            CHECK(update.skipped && fm[k].second.skipped);
            CHECK(update.proj_error == fm[k].second.proj_error);
        }
        CHECK(fm.back().first.root() == fr.root());
    }
    {  // test_metrics.cpp:89-98 / acceptance C5 counting identities
        std::mt19937_64 r5(555555);
        std::vector<Matrix> bases;
        for (Index k = 0; k < 4; ++k) bases.push_back(random_orthonormal(4, 1, r5));
        auto [rep, report] = bht_l2r(tucker_family_batch(bases, 10, r5), DimensionTree::balanced(4), 1e-6);
        CHECK(rep.stored_elements() == 28);
        CHECK(compression_ratio(rep) == 2560.0 / 28.0);
        CHECK(reduction_ratio(rep) == 256.0);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
    return failures ? 1 : 0;
}
