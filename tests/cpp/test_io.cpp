// Container tests against include/htrise/io.hpp, following the reference's
// tests/test_io.cpp cases (round trips, deterministic bytes, normalisation
// metadata, malformed files, corrupt payloads, reload-then-update identity).
//
//   test_io               host-only cases (no GPU needed)
//   test_io --fixtures D  write the deterministic fixtures the Python twin
//                         (paper_2412_16544_b200/io.py) must reproduce byte
//                         for byte
//   test_io --gpu         also the device cases (bht_l2r / ht_rise_update)
#include <htrise/htrise.hpp>
#include <htrise/io.hpp>

#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <random>
#include <string>
#include <vector>

using namespace htrise;
namespace fs = std::filesystem;

namespace {

int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            ++failures;                                                          \
            std::cerr << __FILE__ << ":" << __LINE__ << ": CHECK failed: " #cond "\n"; \
        }                                                                        \
    } while (0)

std::string bytes_of(const std::string& p) {
    std::ifstream f(p, std::ios::binary);
    return {std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>()};
}
void put_bytes(const std::string& p, const std::string& b) {
    std::ofstream f(p, std::ios::binary | std::ios::trunc);
    f.write(b.data(), static_cast<std::streamsize>(b.size()));
}
bool throws_with(const std::function<void()>& fn, const std::string& needle) {
    try {
        fn();
    } catch (const std::runtime_error& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

/// Exactly representable values (dyadic rationals), identical in numpy.
DenseTensor fixture_tensor(const Shape& s, Index salt) {
    DenseTensor t(s);
    for (Index i = 0; i < t.size(); ++i) t.data()[i] = static_cast<double>((i * 7919 + salt * 104729) % 1000 - 500) / 64.0;
    return t;
}

/// A hand-built representation on balanced(3), dims 4x4x4, exactly
/// orthonormal cores (columns of the 4x4 Hadamard matrix / 2).
HTRepresentation fixture_rep() {
    const double h[4][4] = {{1, 1, 1, 1}, {1, -1, 1, -1}, {1, 1, -1, -1}, {1, -1, -1, 1}};
    auto hcols = [&](Shape shape, Index cols) {
        DenseTensor t(shape);
        for (Index c = 0; c < cols; ++c)
            for (Index r = 0; r < 4; ++r) t.data()[r + 4 * c] = 0.5 * h[r][c];
        return t;
    };
    HTRepresentation rep;
    rep.tree = DimensionTree::balanced(3);  // ((1,2),3)
    rep.dims = {4, 4, 4};
    rep.epsilon_rel = 0.2;
    rep.accumulated = 3;
    rep.cores.resize(3);
    rep.cores[0].resize(1);
    rep.cores[1].resize(2);
    rep.cores[2].resize(2);
    // layer 1: transfer (1,0) over leaves (2,0),(2,1) with ranks 2,2 -> 3; leaf (1,1) dim 2 rank 2
    rep.cores[1][0] = hcols({2, 2, 3}, 3);
    rep.cores[1][1] = hcols({4, 2}, 2);
    rep.cores[2][0] = hcols({4, 2}, 2);
    rep.cores[2][1] = hcols({4, 2}, 2);
    rep.cores[0][0] = fixture_tensor({3, 2, 3}, 5);
    return rep;
}

NormalizationParams fixture_norm() {
    NormalizationParams p;
    p.method = NormalizationMethod::ZScore;
    p.field_axis = 1;
    p.scale = {0.2, 1e-05, 100.0, 1e15, 123.456, 0.30000000000000004};
    p.offset = {-0.0, 0.0001, 5e-324, 1.5e+300, -2.5, 1.0 / 3.0};
    p.floored = {false, true, false, false, true, false};
    return p;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "";
    if (mode == "--fixtures") {
        const std::string dir = argc > 2 ? argv[2] : ".";
        fs::create_directories(dir);
        io::write_batch(fixture_tensor({3, 4, 2, 5}, 1), dir + "/batch.bht");
        io::write_batch(fixture_tensor({4, 3, 2}, 2), dir + "/batch_norm.bht", fixture_norm());
        io::RepresentationState st{fixture_rep(), {{1, 3, "y0.bht", fixture_norm()}, {4, 2, "dir/\"q\"\t.bht", {}}}, 2};
        io::write_state(st, dir + "/state.htrs");
        std::cout << "fixtures written\n";
        return 0;
    }

    const fs::path tmp = fs::temp_directory_path() / ("htrise_io_" + std::to_string(std::random_device{}()));
    fs::create_directories(tmp);
    auto file = [&](const std::string& n) { return (tmp / n).string(); };

    {  // JSON number layout of the reference serialiser
        auto d = [](double x) { return json::Value(x).dump(); };
        CHECK(d(0.2) == "0.2");
        CHECK(d(1e-05) == "1e-05");
        CHECK(d(0.0001) == "0.0001");
        CHECK(d(100.0) == "100.0");
        CHECK(d(1e15) == "1e+15");
        CHECK(d(123456789012345.0) == "123456789012345.0");
        CHECK(d(-0.0) == "-0.0");
        CHECK(d(1.5e300) == "1.5e+300");
        CHECK(d(5e-324) == "5e-324");
        CHECK(d(0.1 + 0.2) == "0.30000000000000004");
        CHECK(d(-2.5) == "-2.5");
        json::Value o;
        o["b"] = json::Value::array_of(std::vector<long long>{1, 2});
        o["a"] = "x\"y\\\n\x01";
        CHECK(o.dump() == "{\"a\":\"x\\\"y\\\\\\n\\u0001\",\"b\":[1,2]}");
        const json::Value back = json::Value::parse(o.dump());
        CHECK(back.dump() == o.dump());
        std::mt19937_64 rng(5);
        int bad = 0;
        for (int i = 0; i < 20000; ++i) {  // shortest digits round-trip
            std::uint64_t bits = rng();
            double x;
            std::memcpy(&x, &bits, 8);
            if (!std::isfinite(x)) continue;
            if (json::Value::parse(json::Value(x).dump()).as_double() != x) ++bad;
        }
        CHECK(bad == 0);
    }
    {  // test_io.cpp:42-54 batch round trip, deterministic bytes
        DenseTensor t = fixture_tensor({3, 4, 2, 5}, 3);
        io::write_batch(t, file("batch.bht"));
        DenseTensor back = io::read_batch(file("batch.bht"));
        CHECK(back.shape() == t.shape());
        CHECK(std::memcmp(back.data(), t.data(), sizeof(double) * static_cast<size_t>(t.size())) == 0);
        io::write_batch(t, file("again.bht"));
        CHECK(bytes_of(file("batch.bht")) == bytes_of(file("again.bht")));
    }
    {  // test_io.cpp:56-66 normalisation metadata
        DenseTensor t = fixture_tensor({4, 3, 2}, 4);
        auto [scaled, params] = normalize(t, NormalizationMethod::ZScore, 1);
        io::write_batch(scaled, file("n.bht"), params);
        io::BatchFileContents c = io::read_batch_file(file("n.bht"));
        CHECK(c.normalization.has_value() && *c.normalization == params);
        DenseTensor restored = denormalize(c.tensor, *c.normalization);
        double err = 0.0, nrm = 0.0;
        for (Index i = 0; i < t.size(); ++i) {
            err += (restored.data()[i] - t.data()[i]) * (restored.data()[i] - t.data()[i]);
            nrm += t.data()[i] * t.data()[i];
        }
        CHECK(std::sqrt(err) <= 1e-12 * std::sqrt(nrm));
    }
    {  // test_io.cpp:68-101 malformed batch files
        DenseTensor t = fixture_tensor({2, 3, 2}, 5);
        io::write_batch(t, file("b.bht"));
        const std::string b = bytes_of(file("b.bht"));
        put_bytes(file("short.bht"), b.substr(0, b.size() - 1));
        CHECK(throws_with([&] { io::read_batch(file("short.bht")); }, "truncated"));
        put_bytes(file("long.bht"), b + "x");
        CHECK(throws_with([&] { io::read_batch(file("long.bht")); }, "trailing"));
        std::string bad = b;
        bad[0] = 'X';
        put_bytes(file("magic.bht"), bad);
        CHECK(throws_with([&] { io::read_batch(file("magic.bht")); }, "magic"));
        std::string future = b;
        future[4] = 99;
        put_bytes(file("future.bht"), future);
        CHECK(throws_with([&] { io::read_batch(file("future.bht")); }, "version"));
        CHECK(throws_with([&] { io::read_batch(file("missing.bht")); }, "cannot open"));
        put_bytes(file("tiny.bht"), "BHTB");
        CHECK(throws_with([&] { io::read_batch(file("tiny.bht")); }, "truncated header"));
    }
    {  // test_io.cpp:103-134 state round trip with a ledger
        io::RepresentationState st{fixture_rep(), {{1, 3, "y0.bht", fixture_norm()}}, 1};
        io::write_state(st, file("s.htrs"));
        io::RepresentationState back = io::read_state(file("s.htrs"));
        CHECK(back.rep.tree == st.rep.tree);
        CHECK(back.rep.dims == st.rep.dims);
        CHECK(back.rep.accumulated == st.rep.accumulated);
        CHECK(back.rep.epsilon_rel == st.rep.epsilon_rel);
        CHECK(back.batches_processed == 1);
        CHECK(back.units.size() == 1 && back.units[0] == st.units[0]);
        for (Index l = 0; l <= st.rep.tree.depth(); ++l)
            for (const TreeNode& n : st.rep.tree.layer(l))
                CHECK(back.rep.core(n.id).values() == st.rep.core(n.id).values());
        io::write_state(back, file("s2.htrs"));
        CHECK(bytes_of(file("s.htrs")) == bytes_of(file("s2.htrs")));
    }
    {  // test_io.cpp:181-198 corrupt payload / truncation
        io::write_representation(fixture_rep(), file("r.htrs"));
        std::string b = bytes_of(file("r.htrs"));
        b[b.size() - 9] = static_cast<char>(b[b.size() - 9] ^ 0x41);  // last core: a leaf
        put_bytes(file("corrupt.htrs"), b);
        CHECK(throws_with([&] { io::read_state(file("corrupt.htrs")); }, "corrupt representation"));
        put_bytes(file("trunc.htrs"), b.substr(0, b.size() - 3));
        CHECK(throws_with([&] { io::read_state(file("trunc.htrs")); }, "truncated"));
        HTRepresentation bad = fixture_rep();
        bad.cores[2][0].data()[0] = 2.0;  // not orthonormal: nothing may be written
        CHECK(throws_with([&] { io::write_representation(bad, file("never.htrs")); }, "orthonormality"));
        CHECK(!fs::exists(file("never.htrs")));
    }

    if (mode == "--gpu") {
        std::mt19937_64 rng(61803);
        std::normal_distribution<double> nd;
        auto rnd = [&](Shape s) {
            DenseTensor t(s);
            for (Index i = 0; i < t.size(); ++i) t.data()[i] = nd(rng);
            return t;
        };
        {  // test_io.cpp:152-179 updating a reloaded state matches the in-memory path exactly
            Shape s = {3, 3, 4, 2};
            auto [rep, report] = bht_l2r(rnd(s), DimensionTree::balanced(3), 0.25);
            std::vector<DenseTensor> batches;
            for (int k = 0; k < 3; ++k) batches.push_back(rnd(s));
            HTRepresentation mem = rep;
            for (const DenseTensor& b : batches) mem = ht_rise_update(mem, b).first;
            HTRepresentation disk = rep;
            for (const DenseTensor& b : batches) {
                io::write_representation(disk, file("round.htrs"));
                disk = io::read_representation(file("round.htrs"));
                disk = ht_rise_update(disk, b).first;
            }
            for (Index l = 0; l <= mem.tree.depth(); ++l)
                for (const TreeNode& n : mem.tree.layer(l)) CHECK(disk.core(n.id).values() == mem.core(n.id).values());
        }
        {  // test_io.cpp:136-150 fresh rank-one representation round trip
            DenseTensor y({4, 4, 4, 4, 2});
            for (Index i = 0; i < y.size(); ++i) {
                Index rem = i;
                double v = 1.0;
                for (int k = 0; k < 4; ++k) {
                    v *= 1.0 + static_cast<double>(rem % 4) / (k + 2);
                    rem /= 4;
                }
                y.data()[i] = v * (rem + 1);
            }
            auto [rep, report] = bht_l2r(y, DimensionTree::balanced(4), 1e-6);
            io::write_representation(rep, file("r1.htrs"));
            HTRepresentation back = io::read_representation(file("r1.htrs"));
            for (Index l = 0; l <= rep.tree.depth(); ++l)
                for (const TreeNode& n : rep.tree.layer(l)) CHECK(back.core(n.id).values() == rep.core(n.id).values());
        }
    }

    fs::remove_all(tmp);
    if (failures) {
        std::cout << failures << " FAILED\n";
        return 1;
    }
    std::cout << "ALL PASSED\n";
    return 0;
}
