"""The reference's known-answer tests (tests/golden/reference_kats.json, each
entry citing its source line in the reference's test files) checked against
the CPU oracle, the C++ drop-in headers (host parts) and, on a B200, the
CUDA path. These pin the oracle and the device path to the reference's own
stated answers (the reference cannot be built here: SURVEY 8(c))."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "reference_kats.json")) as f:
    KATS = json.load(f)


def _rank1_batch(dims, batch):
    """test_bht.cpp:19-38: `batch` copies of prod_k v_k[i_k], v_k[i] = 1 + (i + 1)/(k + 2)."""
    grids = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    base = np.ones(dims)
    for k, g in enumerate(grids):
        base = base * (1.0 + (g + 1.0) / (k + 2.0))
    return np.asfortranarray(np.stack([base] * batch, axis=-1))


def _eps_nw_input(kat):
    y = ro.random_tensor(kat["shape"], np.random.default_rng(kat["seed"]))
    return np.asfortranarray(y / np.linalg.norm(y))


def _counting_input(kat):
    rng = np.random.default_rng(kat["seed"])
    bases = [ro.random_orthonormal(n, kat["rank"], rng) for n in kat["dims"]]
    return ro.tucker_family_batch(bases, kat["batch"], rng)


# ---- oracle --------------------------------------------------------------------

@pytest.mark.parametrize("kat", KATS["truncated_svd"], ids=lambda k: k["source"])
def test_oracle_truncated_svd(kat):
    b = ho.truncated_svd(np.array(kat["matrix"], dtype=np.float64), kat["eps"], kat["min_rank"])
    assert b.rank == kat["rank"]
    assert abs(b.discarded_norm - kat["discarded_norm"]) <= kat["tol"]
    if "abs_u" in kat:
        assert np.max(np.abs(np.abs(b.u) - np.array(kat["abs_u"]))) <= kat["tol"]


@pytest.mark.parametrize("kat", KATS["bht_eps_nw"], ids=lambda k: k["source"])
def test_oracle_eps_nw(kat):
    _, rep = ho.bht_l2r(_eps_nw_input(kat), ho.DimensionTree.balanced(kat["d"]), kat["eps"])
    assert abs(rep.eps_nw_initial - kat["eps_nw_initial"]) <= kat["tol"] * kat["eps_nw_initial"]


@pytest.mark.parametrize("kat", KATS["rank1_exact"], ids=lambda k: k["source"])
def test_oracle_rank1_exact(kat):
    y = _rank1_batch(kat["dims"], kat["batch"])
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(len(kat["dims"])), kat["eps"])
    assert set(rep.ranks().values()) == {kat["ranks"]}
    lat, _ = ho.encode(rep, y)
    assert np.linalg.norm(ho.decode(rep, lat) - y) <= kat["rel_err"] * np.linalg.norm(y)


@pytest.mark.parametrize("kat", KATS["counting"], ids=lambda k: k["source"])
def test_oracle_counting(kat):
    rep, _ = ho.bht_l2r(_counting_input(kat), ho.DimensionTree.balanced(len(kat["dims"])), kat["eps"])
    assert rep.stored_elements() == kat["stored_elements"]
    assert abs(ho.compression_ratio(rep) - kat["compression_ratio"]) <= 1e-13 * kat["compression_ratio"]
    if "reduction_ratio" in kat:
        assert ho.reduction_ratio(rep) == kat["reduction_ratio"]


@pytest.mark.parametrize("kat", KATS["pad_with_zeros"], ids=lambda k: k["source"])
def test_oracle_pad_with_zeros(kat):
    core = np.array(kat["core"]).reshape(kat["shape"], order="F")
    out = ho.pad_with_zeros(core, kat["slot"], kat["extra"])
    assert list(out.shape) == kat["padded_shape"]
    assert np.array_equal(out.ravel(order="F"), np.array(kat["padded"]))


@pytest.mark.parametrize("kat", KATS["trees"], ids=lambda k: k["source"])
def test_trees_oracle_and_library(kat):
    from paper_2412_16544_b200 import htrise as ht

    for t in (ho.DimensionTree.balanced(kat["d"]), ht.DimensionTree.balanced(kat["d"])):
        assert t.depth == kat["depth"]
        assert sum(len(layer) for layer in t.layers) == kat["node_count"]
        assert [len(layer) for layer in t.layers] == kat["layer_sizes"]
        for key, dim in kat.get("leaf_dims", {}).items():
            l, p = (int(x) for x in key.split(","))
            assert t.node((l, p)).leaf_dim == dim


# ---- C++ drop-in headers (host parts: normalisation, pad_with_zeros) ------------

def test_cpp_headers_host_kats(tmp_path):
    src = tmp_path / "kats.cpp"
    norm_cases = "".join(
        f'    {{ DenseTensor y({{{len(k["y"])}}}); double v[] = {{{", ".join(map(repr, k["y"]))}}};'
        f' for (int i = 0; i < {len(k["y"])}; ++i) y.data()[i] = v[i];'
        f' auto [s, p] = normalize(y, normalization_from_string("{k["method"]}"));'
        f' out << "{k["source"]}";'
        f' for (Index i = 0; i < s.size(); ++i) out << " " << s.data()[i];'
        f' out << " |"; for (double x : p.scale) out << " " << x; out << " |"; for (double x : p.offset) out << " " << x;'
        f' out << " |"; for (bool b : p.floored) out << " " << b; out << "\\n"; }}\n'
        for k in KATS["normalize"])
    pad = KATS["pad_with_zeros"][0]
    src.write_text(
        "#include <htrise/htrise.hpp>\n#include <iomanip>\n#include <iostream>\n#include <sstream>\n"
        "using namespace htrise;\nint main() {\n  std::ostringstream out; out << std::setprecision(17);\n"
        + norm_cases +
        f'  {{ DenseTensor c({{1, 1, 1}}); c.data()[0] = 1.0; DenseTensor p = pad_with_zeros(c, {pad["slot"]}, {pad["extra"]});'
        ' out << "pad"; for (Index k = 0; k < p.order(); ++k) out << " " << p.extent(k);'
        ' out << " |"; for (Index i = 0; i < p.size(); ++i) out << " " << p.data()[i]; out << "\\n"; }\n'
        "  std::cout << out.str(); return 0;\n}\n")
    exe = tmp_path / "kats"
    from paper_2412_16544_b200 import build
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    str(src), "-L", build.PKG, "-lhtrise_cuda", f"-Wl,-rpath,{build.PKG}", "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines()
    for k, line in zip(KATS["normalize"], lines):
        parts = line.split("|")
        head = parts[0].split()
        assert head[0] == k["source"]
        assert np.allclose([float(x) for x in head[1:]], k["scaled"], rtol=1e-15, atol=0)
        assert [float(x) for x in parts[1].split()] == k["scale"]
        assert [float(x) for x in parts[2].split()] == k["offset"]
        assert [bool(int(x)) for x in parts[3].split()] == k["floored"]
    pad_line = lines[len(KATS["normalize"])].split("|")
    assert [int(x) for x in pad_line[0].split()[1:]] == pad["padded_shape"]
    assert [float(x) for x in pad_line[1].split()] == pad["padded"]


# ---- the CUDA path --------------------------------------------------------------

@pytest.fixture(scope="module")
def ht():
    from paper_2412_16544_b200 import htrise

    htrise.set_default_context(htrise.Context(0))
    return htrise


@pytest.mark.gpu
@pytest.mark.parametrize("kat", KATS["truncated_svd"], ids=lambda k: k["source"])
def test_gpu_truncated_svd(ht, kat):
    b = ht.truncated_svd(np.array(kat["matrix"], dtype=np.float64), kat["eps"], kat["min_rank"])
    assert b.rank == kat["rank"]
    assert abs(b.discarded_norm - kat["discarded_norm"]) <= kat["tol"]
    if "abs_u" in kat:
        assert np.max(np.abs(np.abs(b.u) - np.array(kat["abs_u"]))) <= kat["tol"]


@pytest.mark.gpu
@pytest.mark.parametrize("kat", KATS["bht_eps_nw"], ids=lambda k: k["source"])
def test_gpu_eps_nw(ht, kat):
    _, rep = ht.bht_l2r(_eps_nw_input(kat), ht.DimensionTree.balanced(kat["d"]), kat["eps"])
    assert abs(rep.eps_nw_initial - kat["eps_nw_initial"]) <= kat["tol"] * kat["eps_nw_initial"]


@pytest.mark.gpu
@pytest.mark.parametrize("kat", KATS["rank1_exact"], ids=lambda k: k["source"])
def test_gpu_rank1_exact(ht, kat):
    y = _rank1_batch(kat["dims"], kat["batch"])
    rep, _ = ht.bht_l2r(y, ht.DimensionTree.balanced(len(kat["dims"])), kat["eps"])
    assert set(rep.ranks().values()) == {kat["ranks"]}
    lat, _ = ht.encode(rep, y)
    assert np.linalg.norm(ht.decode(rep, lat) - y) <= kat["rel_err"] * np.linalg.norm(y)


@pytest.mark.gpu
@pytest.mark.parametrize("kat", KATS["counting"], ids=lambda k: k["source"])
def test_gpu_counting(ht, kat):
    rep, _ = ht.bht_l2r(_counting_input(kat), ht.DimensionTree.balanced(len(kat["dims"])), kat["eps"])
    assert rep.stored_elements() == kat["stored_elements"]
    assert abs(ht.compression_ratio(rep) - kat["compression_ratio"]) <= 1e-13 * kat["compression_ratio"]
    if "reduction_ratio" in kat:
        assert ht.reduction_ratio(rep) == kat["reduction_ratio"]
