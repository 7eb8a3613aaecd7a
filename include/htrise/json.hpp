// Minimal JSON value for the HTRS/BHTB container headers (io.hpp).
//
// The reference serialises its headers with nlohmann::json 3.x `dump()`
// (/root/reference/proj/include/htrise/io.hpp:170): objects keep their keys
// sorted (std::map), no whitespace, doubles in shortest round-trip form,
// written in decimal when the decimal point falls within (-4, 15] digits of
// the first digit and as d.ddde+XX otherwise, integral doubles keeping a
// ".0". This writer follows those rules; states written here match the
// reference's byte for byte except that nlohmann prints Grisu2 digits, which
// for ~0.1% of arbitrary doubles differ from the shortest digits in the last
// place (same value either way; tests/cpp/json_pin.cpp pins this against the
// nlohmann copy in the image). The parser accepts any RFC 8259 text.
#pragma once

#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

namespace htrise::json {

class Value;
using Array = std::vector<Value>;
using Object = std::map<std::string, Value>;

class Value {
public:
    using Storage = std::variant<std::nullptr_t, bool, std::int64_t, double, std::string, Array, Object>;

    Value() : v_(nullptr) {}
    Value(std::nullptr_t) : v_(nullptr) {}
    Value(bool b) : v_(b) {}
    Value(int i) : v_(static_cast<std::int64_t>(i)) {}
    Value(long i) : v_(static_cast<std::int64_t>(i)) {}
    Value(long long i) : v_(static_cast<std::int64_t>(i)) {}
    Value(double d) : v_(d) {}
    Value(const char* s) : v_(std::string(s)) {}
    Value(std::string s) : v_(std::move(s)) {}
    Value(Array a) : v_(std::move(a)) {}
    Value(Object o) : v_(std::move(o)) {}
    template <typename T>
    static Value array_of(const std::vector<T>& xs) {
        Array a;
        a.reserve(xs.size());
        for (const T& x : xs) a.emplace_back(x);
        return Value(std::move(a));
    }

    bool is_null() const { return std::holds_alternative<std::nullptr_t>(v_); }
    bool is_int() const { return std::holds_alternative<std::int64_t>(v_); }
    bool is_double() const { return std::holds_alternative<double>(v_); }
    bool is_number() const { return is_int() || is_double(); }
    bool is_string() const { return std::holds_alternative<std::string>(v_); }
    bool is_array() const { return std::holds_alternative<Array>(v_); }
    bool is_object() const { return std::holds_alternative<Object>(v_); }

    std::int64_t as_int() const {
        if (is_int()) return std::get<std::int64_t>(v_);
        if (is_double()) {
            const double d = std::get<double>(v_);
            if (std::floor(d) == d && std::fabs(d) < 9.2e18) return static_cast<std::int64_t>(d);
        }
        throw std::runtime_error("json: expected an integer");
    }
    double as_double() const {
        if (is_double()) return std::get<double>(v_);
        if (is_int()) return static_cast<double>(std::get<std::int64_t>(v_));
        throw std::runtime_error("json: expected a number");
    }
    const std::string& as_string() const {
        if (!is_string()) throw std::runtime_error("json: expected a string");
        return std::get<std::string>(v_);
    }
    const Array& as_array() const {
        if (!is_array()) throw std::runtime_error("json: expected an array");
        return std::get<Array>(v_);
    }
    const Object& as_object() const {
        if (!is_object()) throw std::runtime_error("json: expected an object");
        return std::get<Object>(v_);
    }
    Object& object() {
        if (is_null()) v_ = Object{};
        if (!is_object()) throw std::runtime_error("json: expected an object");
        return std::get<Object>(v_);
    }
    Value& operator[](const std::string& key) { return object()[key]; }
    const Value& at(const std::string& key) const {
        const Object& o = as_object();
        auto it = o.find(key);
        if (it == o.end()) throw std::runtime_error("json: missing key \"" + key + "\"");
        return it->second;
    }
    const Value& at(std::size_t i) const {
        const Array& a = as_array();
        if (i >= a.size()) throw std::runtime_error("json: array index out of range");
        return a[i];
    }
    bool contains(const std::string& key) const { return is_object() && as_object().count(key) > 0; }
    std::vector<std::int64_t> as_int_vector() const {
        std::vector<std::int64_t> out;
        for (const Value& x : as_array()) out.push_back(x.as_int());
        return out;
    }
    std::vector<double> as_double_vector() const {
        std::vector<double> out;
        for (const Value& x : as_array()) out.push_back(x.as_double());
        return out;
    }

    std::string dump() const {
        std::string out;
        write(out);
        return out;
    }
    /// Pretty form (nlohmann's dump(indent) layout: one member per line,
    /// "key": value, empty containers inline).
    std::string dump(int indent) const {
        std::string out;
        write_pretty(out, indent, 0);
        return out;
    }
    void write(std::string& out) const;
    void write_pretty(std::string& out, int indent, int level) const;
    static Value parse(const char* first, const char* last);
    static Value parse(const std::string& s) { return parse(s.data(), s.data() + s.size()); }

private:
    Storage v_;
};

namespace detail {

/// nlohmann's float layout over the shortest round-trip digits.
inline void write_double(std::string& out, double v) {
    if (!std::isfinite(v)) {
        out += "null";
        return;
    }
    if (v == 0.0) {
        out += std::signbit(v) ? "-0.0" : "0.0";
        return;
    }
    char sci[64];
    auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
    std::string s(sci, r.ptr);
    std::string sign;
    if (s[0] == '-') {
        sign = "-";
        s.erase(0, 1);
    }
    const std::size_t e_pos = s.find('e');
    const int exp10 = std::stoi(s.substr(e_pos + 1));
    std::string digits;
    for (std::size_t i = 0; i < e_pos; ++i)
        if (s[i] != '.') digits.push_back(s[i]);
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // decimal point position relative to the first digit
    constexpr int kMinExp = -4, kMaxExp = 15;
    out += sign;
    if (k <= n && n <= kMaxExp) {
        out += digits;
        out.append(static_cast<std::size_t>(n - k), '0');
        out += ".0";
    } else if (0 < n && n <= kMaxExp) {
        out += digits.substr(0, static_cast<std::size_t>(n));
        out += '.';
        out += digits.substr(static_cast<std::size_t>(n));
    } else if (kMinExp < n && n <= 0) {
        out += "0.";
        out.append(static_cast<std::size_t>(-n), '0');
        out += digits;
    } else {
        out += digits[0];
        if (k > 1) {
            out += '.';
            out += digits.substr(1);
        }
        int e = n - 1;
        out += 'e';
        out += e < 0 ? '-' : '+';
        e = e < 0 ? -e : e;
        if (e < 10) out += '0';
        out += std::to_string(e);
    }
}

inline void write_string(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof(buf), "\\u%04x", static_cast<unsigned>(c));
                    out += buf;
                } else {
                    out += static_cast<char>(c);
                }
        }
    }
    out += '"';
}

class Parser {
public:
    Parser(const char* first, const char* last) : p_(first), end_(last) {}

    Value document() {
        Value v = value();
        ws();
        if (p_ != end_) fail("trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const std::string& what) const { throw std::runtime_error("json parse error: " + what); }
    void ws() {
        while (p_ != end_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* s) {
        const std::size_t n = std::strlen(s);
        if (static_cast<std::size_t>(end_ - p_) >= n && std::memcmp(p_, s, n) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }
    Value value() {
        ws();
        if (p_ == end_) fail("unexpected end");
        switch (*p_) {
            case '{': return object();
            case '[': return array();
            case '"': return Value(string());
            case 't': if (lit("true")) return Value(true); break;
            case 'f': if (lit("false")) return Value(false); break;
            case 'n': if (lit("null")) return Value(nullptr); break;
            default: return number();
        }
        fail("invalid literal");
    }
    Value object() {
        ++p_;
        Object o;
        ws();
        if (p_ != end_ && *p_ == '}') {
            ++p_;
            return Value(std::move(o));
        }
        for (;;) {
            ws();
            if (p_ == end_ || *p_ != '"') fail("expected a key");
            std::string k = string();
            ws();
            if (p_ == end_ || *p_ != ':') fail("expected ':'");
            ++p_;
            o[std::move(k)] = value();
            ws();
            if (p_ != end_ && *p_ == ',') {
                ++p_;
                continue;
            }
            if (p_ != end_ && *p_ == '}') {
                ++p_;
                return Value(std::move(o));
            }
            fail("expected ',' or '}'");
        }
    }
    Value array() {
        ++p_;
        Array a;
        ws();
        if (p_ != end_ && *p_ == ']') {
            ++p_;
            return Value(std::move(a));
        }
        for (;;) {
            a.push_back(value());
            ws();
            if (p_ != end_ && *p_ == ',') {
                ++p_;
                continue;
            }
            if (p_ != end_ && *p_ == ']') {
                ++p_;
                return Value(std::move(a));
            }
            fail("expected ',' or ']'");
        }
    }
    static void put_utf8(std::string& s, std::uint32_t cp) {
        if (cp < 0x80) {
            s += static_cast<char>(cp);
        } else if (cp < 0x800) {
            s += static_cast<char>(0xC0 | (cp >> 6));
            s += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            s += static_cast<char>(0xE0 | (cp >> 12));
            s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            s += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            s += static_cast<char>(0xF0 | (cp >> 18));
            s += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            s += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    std::uint32_t hex4() {
        if (end_ - p_ < 4) fail("short \\u escape");
        std::uint32_t v = 0;
        for (int i = 0; i < 4; ++i, ++p_) {
            const char c = *p_;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<std::uint32_t>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<std::uint32_t>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<std::uint32_t>(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        ++p_;
        std::string s;
        for (;;) {
            if (p_ == end_) fail("unterminated string");
            const char c = *p_++;
            if (c == '"') return s;
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
            if (c != '\\') {
                s += c;
                continue;
            }
            if (p_ == end_) fail("unterminated escape");
            const char e = *p_++;
            switch (e) {
                case '"': s += '"'; break;
                case '\\': s += '\\'; break;
                case '/': s += '/'; break;
                case 'b': s += '\b'; break;
                case 'f': s += '\f'; break;
                case 'n': s += '\n'; break;
                case 'r': s += '\r'; break;
                case 't': s += '\t'; break;
                case 'u': {
                    std::uint32_t cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00) {
                        if (!lit("\\u")) fail("unpaired surrogate");
                        const std::uint32_t lo = hex4();
                        if (lo < 0xDC00 || lo >= 0xE000) fail("bad surrogate pair");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    put_utf8(s, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
    }
    Value number() {
        const char* start = p_;
        if (p_ != end_ && *p_ == '-') ++p_;
        if (p_ == end_ || !(*p_ >= '0' && *p_ <= '9')) fail("invalid number");
        if (*p_ == '0') ++p_;
        else
            while (p_ != end_ && *p_ >= '0' && *p_ <= '9') ++p_;
        bool is_float = false;
        if (p_ != end_ && *p_ == '.') {
            is_float = true;
            ++p_;
            if (p_ == end_ || !(*p_ >= '0' && *p_ <= '9')) fail("invalid fraction");
            while (p_ != end_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (p_ != end_ && (*p_ == 'e' || *p_ == 'E')) {
            is_float = true;
            ++p_;
            if (p_ != end_ && (*p_ == '+' || *p_ == '-')) ++p_;
            if (p_ == end_ || !(*p_ >= '0' && *p_ <= '9')) fail("invalid exponent");
            while (p_ != end_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (!is_float) {
            std::int64_t i = 0;
            auto r = std::from_chars(start, p_, i);
            if (r.ec == std::errc() && r.ptr == p_) return Value(i);
        }
        double d = 0.0;
        auto r = std::from_chars(start, p_, d);
        if (r.ec != std::errc() || r.ptr != p_) fail("invalid number");
        return Value(d);
    }

    const char* p_;
    const char* end_;
};

}  // namespace detail

inline void Value::write(std::string& out) const {
    switch (v_.index()) {
        case 0: out += "null"; break;
        case 1: out += std::get<bool>(v_) ? "true" : "false"; break;
        case 2: out += std::to_string(std::get<std::int64_t>(v_)); break;
        case 3: detail::write_double(out, std::get<double>(v_)); break;
        case 4: detail::write_string(out, std::get<std::string>(v_)); break;
        case 5: {
            out += '[';
            bool first = true;
            for (const Value& x : std::get<Array>(v_)) {
                if (!first) out += ',';
                first = false;
                x.write(out);
            }
            out += ']';
            break;
        }
        default: {
            out += '{';
            bool first = true;
            for (const auto& [k, x] : std::get<Object>(v_)) {
                if (!first) out += ',';
                first = false;
                detail::write_string(out, k);
                out += ':';
                x.write(out);
            }
            out += '}';
        }
    }
}

inline void Value::write_pretty(std::string& out, int indent, int level) const {
    const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
    const std::string close(static_cast<std::size_t>(indent * level), ' ');
    if (is_array() && !as_array().empty()) {
        out += "[\n";
        bool first = true;
        for (const Value& x : as_array()) {
            if (!first) out += ",\n";
            first = false;
            out += pad;
            x.write_pretty(out, indent, level + 1);
        }
        out += "\n" + close + "]";
    } else if (is_object() && !as_object().empty()) {
        out += "{\n";
        bool first = true;
        for (const auto& [k, x] : as_object()) {
            if (!first) out += ",\n";
            first = false;
            out += pad;
            detail::write_string(out, k);
            out += ": ";
            x.write_pretty(out, indent, level + 1);
        }
        out += "\n" + close + "}";
    } else {
        write(out);
    }
}

inline Value Value::parse(const char* first, const char* last) { return detail::Parser(first, last).document(); }

}  // namespace htrise::json
