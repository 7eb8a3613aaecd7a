"""BHTB / HTRS containers (reference io.hpp; tests follow its test_io.cpp and
acceptance criterion C9): the C++ drop-in (include/htrise/io.hpp), its Python
twin (paper_2412_16544_b200/io.py), byte identity between the two, the
header serialiser pinned to nlohmann::json, and (GPU) resuming a stream
from a state file reproducing the uninterrupted run bit for bit."""
import os
import subprocess

import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro
from paper_2412_16544_b200 import build
from paper_2412_16544_b200 import io


@pytest.fixture(scope="module")
def io_bin():
    return build.build_io_test()


def test_cpp_container_cases_host(io_bin):
    r = subprocess.run([io_bin], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr


def test_header_serialiser_pinned_to_nlohmann():
    pin = build.build_json_pin()
    if pin is None:
        pytest.skip("nlohmann::json header not present in this image")
    r = subprocess.run([pin], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    emitted = subprocess.run([pin, "--emit"], capture_output=True, text=True, timeout=60).stdout.split()
    curated = [0.2, 1e-05, 0.0001, 100.0, 1e15, 1e16, 123456789012345.0, 1234567890123456.0, -0.0, 0.0, 1.5e300,
               5e-324, 0.1 + 0.2, -2.5, 1.0 / 3.0, 2.0 / 3.0, 1e-3, 9.999999999999999e-5, 0.00012345, 1e21, 1e22, 4.35,
               0.3, 2.2250738585072014e-308, 1.7976931348623157e308, 3.0, 1e-14, 0.25, 0.125]
    for x, want in zip(curated, emitted):
        assert io.dump_json(x) == want, (x, want)
    for e, want in zip(range(-320, 309), emitted[len(curated):]):
        x = 10.0 ** e if e > -308 else float(want)
        ours = io.dump_json(x)
        assert ours == want or float(ours) == float(want) == x, (e, ours, want)


def _fixture_tensor(shape, salt):
    n = int(np.prod(shape))
    i = np.arange(n, dtype=np.int64)
    v = ((i * 7919 + salt * 104729) % 1000 - 500) / 64.0
    return v.reshape(shape, order="F")


def _fixture_norm():
    return io.NormalizationParams("zscore", 1, [0.2, 1e-05, 100.0, 1e15, 123.456, 0.30000000000000004],
                                  [-0.0, 0.0001, 5e-324, 1.5e300, -2.5, 1.0 / 3.0],
                                  [False, True, False, False, True, False])


def _fixture_rep():
    from paper_2412_16544_b200 import htrise as ht

    h = 0.5 * np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], dtype=np.float64)
    cores = {(1, 0): h[:, :3].reshape((2, 2, 3), order="F"), (1, 1): h[:, :2].copy(), (2, 0): h[:, :2].copy(),
             (2, 1): h[:, :2].copy(), (0, 0): _fixture_tensor((3, 2, 3), 5)}
    return io.HostRepresentation(ht.DimensionTree.balanced(3), [4, 4, 4], cores, 3, 0.2)


def test_python_twin_writes_the_same_bytes(io_bin, tmp_path):
    cpp = tmp_path / "cpp"
    r = subprocess.run([io_bin, "--fixtures", str(cpp)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    py = tmp_path / "py"
    py.mkdir()
    io.write_batch(_fixture_tensor((3, 4, 2, 5), 1), str(py / "batch.bht"))
    io.write_batch(_fixture_tensor((4, 3, 2), 2), str(py / "batch_norm.bht"), _fixture_norm())
    state = io.RepresentationState(_fixture_rep(), [io.UnitRecord(1, 3, "y0.bht", _fixture_norm()),
                                                    io.UnitRecord(4, 2, 'dir/"q"\t.bht', io.NormalizationParams())], 2)
    io.write_state(state, str(py / "state.htrs"))
    for name in ("batch.bht", "batch_norm.bht", "state.htrs"):
        assert (cpp / name).read_bytes() == (py / name).read_bytes(), name
    # and the Python reader takes the C++ file back exactly
    back = io.read_state(str(cpp / "state.htrs"), device=False)
    assert back.batches_processed == 2 and back.units == state.units
    for nid, c in _fixture_rep().cores.items():
        assert np.array_equal(back.rep.core(nid), c)


def test_batch_round_trip_and_malformed(tmp_path):
    rng = np.random.default_rng(61803)
    t = np.asfortranarray(rng.standard_normal((3, 4, 2, 5)))
    p = str(tmp_path / "b.bht")
    io.write_batch(t, p)
    back, norm = io.read_batch_file(p)
    assert norm is None and back.shape == t.shape and np.array_equal(back, t)
    io.write_batch(t, str(tmp_path / "again.bht"))
    assert (tmp_path / "again.bht").read_bytes() == open(p, "rb").read()
    b = open(p, "rb").read()
    cases = {"short": (b[:-1], "truncated"), "long": (b + b"x", "trailing"), "magic": (b"X" + b[1:], "magic"),
             "future": (b[:4] + bytes([99]) + b[5:], "version"), "tiny": (b"BHTB", "truncated header")}
    for name, (data, needle) in cases.items():
        q = tmp_path / f"{name}.bht"
        q.write_bytes(data)
        with pytest.raises(RuntimeError, match=needle):
            io.read_batch(str(q))
    with pytest.raises(RuntimeError, match="cannot open"):
        io.read_batch(str(tmp_path / "missing.bht"))


def test_state_round_trip_of_an_oracle_representation(tmp_path):
    rng = np.random.default_rng(7)
    y = ro.random_tensor([3, 4, 3, 3], rng)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.2)
    unit = io.UnitRecord(1, 3, "y0.bht", io.NormalizationParams("maxabs", None, [float(np.max(np.abs(y)))], [0.0],
                                                                [False]))
    p = str(tmp_path / "s.htrs")
    io.write_state(io.RepresentationState(rep, [unit], 1), p)
    back = io.read_state(p, device=False)
    assert back.rep.dims == rep.dims and back.rep.accumulated == rep.accumulated
    assert back.rep.epsilon_rel == rep.epsilon_rel and back.batches_processed == 1 and back.units == [unit]
    for l in range(rep.tree.depth + 1):
        for n in rep.tree.layer(l):
            assert np.array_equal(back.rep.core(n.id), rep.core(n.id))
    p2 = str(tmp_path / "s2.htrs")
    io.write_state(back, p2)
    assert open(p, "rb").read() == open(p2, "rb").read()
    # a corrupted leaf fails the invariant checks on read; a truncated file too
    b = bytearray(open(p, "rb").read())
    b[-9] ^= 0x41
    (tmp_path / "c.htrs").write_bytes(bytes(b))
    with pytest.raises(RuntimeError, match="corrupt representation"):
        io.read_state(str(tmp_path / "c.htrs"), device=False)
    (tmp_path / "t.htrs").write_bytes(bytes(b[:-3]))
    with pytest.raises(RuntimeError, match="truncated"):
        io.read_state(str(tmp_path / "t.htrs"), device=False)


@pytest.mark.gpu
def test_cpp_container_cases_gpu(io_bin):
    r = subprocess.run([io_bin, "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_resumed_stream_matches_uninterrupted_run(tmp_path):
    """test_io.cpp:152-179 / acceptance C9 on the device path: write the
    state after every batch, read it back into HBM, continue; the cores and
    the final state file equal the uninterrupted run's bit for bit (fused
    skip path and expansions included)."""
    from paper_2412_16544_b200 import htrise as ht

    ht.set_default_context(ht.Context(0))
    rng = np.random.default_rng(99)
    bases = [ro.random_orthonormal(64, 4, rng) for _ in range(3)]
    wide = [np.hstack([b, ro.random_orthonormal(64, 2, rng)]) for b in bases]
    batches = [ro.tucker_family_batch(bases, 6, rng) + 1e-9 * rng.standard_normal((64, 64, 64, 6))
               for _ in range(3)]
    batches.append(ro.tucker_family_batch(wide, 5, rng))
    batches.append(ro.tucker_family_batch(bases, 4, rng))
    mem, _ = ht.bht_l2r(batches[0], ht.tree_1_23(), 1e-3)
    disk = mem
    p = str(tmp_path / "round.htrs")
    for k, b in enumerate(batches[1:]):
        mem, um = ht.ht_rise_update(mem, b)
        io.write_state(io.RepresentationState(disk, [], k + 1), p)
        disk = io.read_state(p).rep
        disk, ud = ht.ht_rise_update(disk, b)
        assert um.skipped == ud.skipped and um.proj_error == ud.proj_error
    for l in range(mem.tree.depth + 1):
        for n in mem.tree.layer(l):
            assert np.array_equal(disk.core(n.id), mem.core(n.id)), n.id
    io.write_representation(mem, str(tmp_path / "a.htrs"))
    io.write_representation(disk, str(tmp_path / "b.htrs"))
    assert (tmp_path / "a.htrs").read_bytes() == (tmp_path / "b.htrs").read_bytes()
