// htrise-b200 drop-in: BHTB batch and HTRS state containers (reference
// /root/reference/proj/include/htrise/io.hpp: format constants 23-25,
// UnitRecord 29-36, RepresentationState 40-44, container layout 166-180,
// write_batch 208-217, read_batch_file 224-239, read_batch 241-243,
// write_state 249-299, read_state 301-387, write/read_representation 390-396).
//
// Layout: 4-byte magic, u16 format version (1), u32 header length, the
// header as compact JSON (json.hpp reproduces the reference's serialiser),
// then little-endian f64 payload. A state's payload is every core, layer
// major and position minor, root included. Writing the same state twice
// gives the same bytes; against the reference's writer only header doubles
// can differ, in the last printed digit (json.hpp). For a device-resident
// representation the cores are exported
// from HBM exactly (fetch_core) and a read state is re-imported on first use,
// so updating a reloaded state reproduces the in-memory stream bit for bit.
#pragma once

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "htrise/bht.hpp"
#include "htrise/json.hpp"
#include "htrise/metrics.hpp"

namespace htrise::io {

inline constexpr std::uint16_t kFormatVersion = 1;
inline constexpr char kBatchMagic[4] = {'B', 'H', 'T', 'B'};
inline constexpr char kStateMagic[4] = {'H', 'T', 'R', 'S'};

/// One streamed unit of the normalisation ledger.
struct UnitRecord {
    Index first = 0;  ///< 1-based index of the unit's first tensor
    Index count = 0;
    std::string source;
    NormalizationParams norm;

    bool operator==(const UnitRecord&) const = default;
};

/// Representation plus the CLI's ledger and batch counter.
struct RepresentationState {
    HTRepresentation rep;
    std::vector<UnitRecord> units;
    Index batches_processed = 0;
};

struct BatchFileContents {
    DenseTensor tensor;
    std::optional<NormalizationParams> normalization;
};

namespace detail {

inline void append_le(std::string& out, std::uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xffu));
}

inline void append_f64(std::string& out, const double* v, Index n) {
    const std::size_t at = out.size();
    out.resize(at + static_cast<std::size_t>(n) * 8);
    for (Index i = 0; i < n; ++i) {
        std::uint64_t bits;
        std::memcpy(&bits, v + i, 8);
        for (int b = 0; b < 8; ++b)
            out[at + static_cast<std::size_t>(i) * 8 + static_cast<std::size_t>(b)] =
                static_cast<char>((bits >> (8 * b)) & 0xffu);
    }
}

inline std::string container(const char magic[4], const json::Value& header,
                             const std::vector<const DenseTensor*>& payload) {
    const std::string h = header.dump();
    Index total = 0;
    for (const DenseTensor* t : payload) total += t->size();
    std::string out(magic, 4);
    out.reserve(10 + h.size() + static_cast<std::size_t>(total) * 8);
    append_le(out, kFormatVersion, 2);
    append_le(out, static_cast<std::uint32_t>(h.size()), 4);
    out += h;
    for (const DenseTensor* t : payload) append_f64(out, t->data(), t->size());
    return out;
}

/// Atomic publication: a sibling temporary, then rename.
inline void publish(const std::string& path, const std::string& bytes) {
    const std::string tmp = path + ".tmp";
    {
        std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
        if (!f) throw std::runtime_error(tmp + ": cannot open for writing");
        f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
        if (!f) throw std::runtime_error(tmp + ": write failed");
    }
    std::filesystem::rename(tmp, path);
}

/// Container reader: validates magic, version and header bounds.
class Container {
public:
    Container(const std::string& path, const char magic[4]) : path_(path) {
        std::ifstream f(path, std::ios::binary);
        if (!f) throw std::runtime_error(path + ": cannot open");
        bytes_.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
        if (bytes_.size() < 10) throw std::runtime_error(path + ": truncated header");
        if (std::memcmp(bytes_.data(), magic, 4) != 0) throw std::runtime_error(path + ": bad magic");
        pos_ = 4;
        const auto version = static_cast<std::uint16_t>(le(2));
        if (version > kFormatVersion)
            throw std::runtime_error(path + ": unsupported format version " + std::to_string(version));
        const std::uint64_t hlen = le(4);
        if (bytes_.size() - pos_ < hlen) throw std::runtime_error(path + ": truncated header");
        try {
            header_ = json::Value::parse(bytes_.data() + pos_, bytes_.data() + pos_ + hlen);
        } catch (const std::exception& e) {
            throw std::runtime_error(path + ": corrupt header: " + e.what());
        }
        pos_ += hlen;
    }
    const json::Value& header() const { return header_; }
    const std::string& path() const { return path_; }

    Vector payload(Index n) {
        if (n < 0 || (bytes_.size() - pos_) / 8 < static_cast<std::size_t>(n))
            throw std::runtime_error(path_ + ": truncated payload");
        Vector v(n);
        for (Index i = 0; i < n; ++i) {
            std::uint64_t bits = 0;
            for (int b = 0; b < 8; ++b)
                bits |= static_cast<std::uint64_t>(static_cast<unsigned char>(bytes_[pos_ + static_cast<std::size_t>(b)]))
                        << (8 * b);
            std::memcpy(&v[i], &bits, 8);
            pos_ += 8;
        }
        return v;
    }
    void expect_end() const {
        if (pos_ != bytes_.size()) throw std::runtime_error(path_ + ": trailing bytes after payload");
    }

private:
    std::uint64_t le(int n) {
        std::uint64_t v = 0;
        for (int i = 0; i < n; ++i)
            v |= static_cast<std::uint64_t>(static_cast<unsigned char>(bytes_[pos_ + static_cast<std::size_t>(i)]))
                 << (8 * i);
        pos_ += static_cast<std::size_t>(n);
        return v;
    }

    std::string path_;
    std::string bytes_;
    std::size_t pos_ = 0;
    json::Value header_;
};

inline json::Value norm_json(const NormalizationParams& p) {
    json::Value j;
    j["method"] = to_string(p.method);
    if (p.field_axis) j["field_axis"] = static_cast<long long>(*p.field_axis);
    j["scale"] = json::Value::array_of(p.scale);
    j["offset"] = json::Value::array_of(p.offset);
    json::Array fl;
    for (bool b : p.floored) fl.emplace_back(b ? 1 : 0);
    j["floored"] = json::Value(std::move(fl));
    return j;
}

inline NormalizationParams norm_from(const json::Value& j) {
    NormalizationParams p;
    p.method = normalization_from_string(j.at("method").as_string());
    if (j.contains("field_axis")) p.field_axis = j.at("field_axis").as_int();
    p.scale = j.at("scale").as_double_vector();
    p.offset = j.at("offset").as_double_vector();
    for (std::int64_t b : j.at("floored").as_int_vector()) p.floored.push_back(b != 0);
    return p;
}

inline json::Value shape_json(const Shape& s) {
    json::Array a;
    for (Index x : s) a.emplace_back(static_cast<long long>(x));
    return json::Value(std::move(a));
}

inline Shape shape_from(const json::Value& j) {
    Shape s;
    for (std::int64_t x : j.as_int_vector()) s.push_back(x);
    return s;
}

inline json::Value id_json(NodeId id) {
    return json::Value(json::Array{json::Value(static_cast<long long>(id.layer)), json::Value(static_cast<long long>(id.pos))});
}

}  // namespace detail

/// Batch container: canonical-order f64 payload, shape with the batch axis last.
inline void write_batch(const DenseTensor& t, const std::string& path,
                        const std::optional<NormalizationParams>& norm = std::nullopt) {
    json::Value h;
    h["dtype"] = "f64";
    h["layout"] = "first-fastest";
    h["shape"] = detail::shape_json(t.shape());
    if (norm) h["normalization"] = detail::norm_json(*norm);
    detail::publish(path, detail::container(kBatchMagic, h, {&t}));
}

inline BatchFileContents read_batch_file(const std::string& path) {
    detail::Container r(path, kBatchMagic);
    const json::Value& h = r.header();
    try {
        if (h.at("dtype").as_string() != "f64" || h.at("layout").as_string() != "first-fastest")
            throw std::runtime_error(path + ": unsupported dtype or layout");
        Shape shape = detail::shape_from(h.at("shape"));
        BatchFileContents out{DenseTensor(shape, r.payload(shape_product(shape))), std::nullopt};
        r.expect_end();
        if (h.contains("normalization")) out.normalization = detail::norm_from(h.at("normalization"));
        return out;
    } catch (const std::invalid_argument& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
}

inline DenseTensor read_batch(const std::string& path) { return read_batch_file(path).tensor; }

/// Persist a representation with its ledger. The representation invariants
/// are checked before anything touches the disk.
inline void write_state(const RepresentationState& state, const std::string& path) {
    const HTRepresentation& rep = state.rep;
    rep.validate();
    json::Value h;
    h["dims"] = detail::shape_json(rep.dims);
    h["epsilon_rel"] = rep.epsilon_rel;
    h["accumulated"] = static_cast<long long>(rep.accumulated);
    h["batches_processed"] = static_cast<long long>(state.batches_processed);
    json::Array nodes, shapes;
    std::vector<const DenseTensor*> payload;
    for (Index l = 0; l <= rep.tree.depth(); ++l)
        for (const TreeNode& n : rep.tree.layer(l)) {
            json::Value jn;
            jn["layer"] = static_cast<long long>(n.id.layer);
            jn["pos"] = static_cast<long long>(n.id.pos);
            jn["kind"] = n.kind == NodeKind::Root ? "root" : n.kind == NodeKind::Transfer ? "transfer" : "leaf";
            if (n.kind == NodeKind::Leaf) {
                jn["leaf_dim"] = static_cast<long long>(n.leaf_dim);
            } else {
                jn["successors"] = json::Value(json::Array{detail::id_json(n.successors[0]), detail::id_json(n.successors[1])});
            }
            if (n.kind != NodeKind::Root) jn["parent"] = detail::id_json(n.parent);
            nodes.push_back(std::move(jn));
            const DenseTensor& c = rep.core(n.id);
            shapes.push_back(detail::shape_json(c.shape()));
            payload.push_back(&c);
        }
    json::Value tree;
    tree["d"] = static_cast<long long>(rep.tree.dims());
    tree["nodes"] = json::Value(std::move(nodes));
    h["tree"] = std::move(tree);
    h["core_shapes"] = json::Value(std::move(shapes));
    json::Array units;
    for (const UnitRecord& u : state.units) {
        json::Value ju;
        ju["first"] = static_cast<long long>(u.first);
        ju["count"] = static_cast<long long>(u.count);
        ju["source"] = u.source;
        ju["norm"] = detail::norm_json(u.norm);
        units.push_back(std::move(ju));
    }
    h["units"] = json::Value(std::move(units));
    detail::publish(path, detail::container(kStateMagic, h, payload));
}

inline RepresentationState read_state(const std::string& path) {
    detail::Container r(path, kStateMagic);
    const json::Value& h = r.header();
    RepresentationState state;
    HTRepresentation& rep = state.rep;
    const json::Value& jtree = h.at("tree");
    std::vector<std::vector<TreeNode>> layers;
    for (const json::Value& jn : jtree.at("nodes").as_array()) {
        TreeNode n;
        n.id = {jn.at("layer").as_int(), jn.at("pos").as_int()};
        const std::string& kind = jn.at("kind").as_string();
        if (kind == "root") n.kind = NodeKind::Root;
        else if (kind == "transfer") n.kind = NodeKind::Transfer;
        else if (kind == "leaf") n.kind = NodeKind::Leaf;
        else throw std::runtime_error(path + ": unknown node kind " + kind);
        if (n.kind == NodeKind::Leaf) {
            n.leaf_dim = jn.at("leaf_dim").as_int();
        } else {
            for (const json::Value& js : jn.at("successors").as_array())
                n.successors.push_back({js.at(std::size_t{0}).as_int(), js.at(std::size_t{1}).as_int()});
        }
        if (n.id.layer < 0 || n.id.pos < 0) throw std::runtime_error(path + ": node records out of order");
        if (static_cast<std::size_t>(n.id.layer) >= layers.size()) layers.resize(static_cast<std::size_t>(n.id.layer) + 1);
        auto& layer = layers[static_cast<std::size_t>(n.id.layer)];
        if (static_cast<Index>(layer.size()) != n.id.pos) throw std::runtime_error(path + ": node records out of order");
        layer.push_back(std::move(n));
    }
    try {
        rep.tree = DimensionTree::from_layers(std::move(layers));
    } catch (const std::invalid_argument& e) {
        throw std::runtime_error(path + ": corrupt tree: " + e.what());
    }
    if (rep.tree.dims() != jtree.at("d").as_int()) throw std::runtime_error(path + ": tree dimension mismatch");
    for (const json::Value& jn : jtree.at("nodes").as_array()) {
        const NodeId id{jn.at("layer").as_int(), jn.at("pos").as_int()};
        if (id.layer == 0) continue;
        const json::Value& jp = jn.at("parent");
        const NodeId parent{jp.at(std::size_t{0}).as_int(), jp.at(std::size_t{1}).as_int()};
        if (rep.tree.node(id).parent != parent)
            throw std::runtime_error(path + ": corrupt parent link at node " + to_string(id));
    }
    rep.dims = detail::shape_from(h.at("dims"));
    rep.epsilon_rel = h.at("epsilon_rel").as_double();
    rep.accumulated = h.at("accumulated").as_int();
    state.batches_processed = h.at("batches_processed").as_int();
    const json::Array& jshapes = h.at("core_shapes").as_array();
    rep.cores.assign(static_cast<std::size_t>(rep.tree.depth()) + 1, {});
    std::size_t k = 0;
    for (Index l = 0; l <= rep.tree.depth(); ++l)
        for (Index i = 0; i < rep.tree.layer_size(l); ++i, ++k) {
            if (k >= jshapes.size()) throw std::runtime_error(path + ": missing core shape");
            Shape s = detail::shape_from(jshapes[k]);
            rep.cores[static_cast<std::size_t>(l)].emplace_back(s, r.payload(shape_product(s)));
        }
    r.expect_end();
    for (const json::Value& ju : h.at("units").as_array()) {
        UnitRecord u;
        u.first = ju.at("first").as_int();
        u.count = ju.at("count").as_int();
        u.source = ju.at("source").as_string();
        u.norm = detail::norm_from(ju.at("norm"));
        state.units.push_back(std::move(u));
    }
    try {
        rep.validate();
    } catch (const std::exception& e) {
        throw std::runtime_error(path + ": corrupt representation: " + e.what());
    }
    return state;
}

/// Bare representation, no ledger.
inline void write_representation(const HTRepresentation& h, const std::string& path) {
    write_state(RepresentationState{h, {}, 0}, path);
}

inline HTRepresentation read_representation(const std::string& path) { return read_state(path).rep; }

}  // namespace htrise::io
