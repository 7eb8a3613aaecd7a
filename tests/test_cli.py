"""The `htrise` command-line tool (reference tools/main.cpp), following the
reference's tests/test_cli.cpp and acceptance criterion C9. Compression
runs on the GPU; usage errors and `inspect` of a state written on the host
run here."""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro
from paper_2412_16544_b200 import build
from paper_2412_16544_b200 import io


@pytest.fixture(scope="module")
def cli():
    return build.build_cli()


def run(cli, *args):
    r = subprocess.run([cli, *[str(a) for a in args]], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


def rows(path):
    with open(path) as f:
        return list(csv.reader(f))


def test_usage_errors(cli, tmp_path):
    assert run(cli)[0] == 106
    rc, out = run(cli, "compress", tmp_path / "a.bht", "--epsilon", "1.5", "--state", tmp_path / "s.htrs")
    assert rc == 106 and "range" in out
    rc, out = run(cli, "compress", tmp_path / "a.bht", "--state", tmp_path / "s.htrs")
    assert rc == 106 and "--epsilon" in out
    rc, out = run(cli, "compress", tmp_path / "a.bht", "--epsilon", "0.1", "--state", tmp_path / "s.htrs",
                  "--normalize", "median")
    assert rc == 106
    rc, out = run(cli, "decode", "--state", tmp_path / "s.htrs", "--out", tmp_path / "o.bht")
    assert rc == 1 and "exactly one" in out
    assert run(cli, "--help")[0] == 0


def test_inspect_host_state(cli, tmp_path):
    rng = np.random.default_rng(3)
    rep, _ = ho.bht_l2r(ro.random_tensor([3, 3, 3, 3, 2], rng), ho.DimensionTree.balanced(4), 0.2)
    p = tmp_path / "s.htrs"
    io.write_state(io.RepresentationState(rep, [], 1), str(p))
    rc, out = run(cli, "inspect", "--state", p)
    assert rc == 0 and "7 nodes" in out, out
    rc, out = run(cli, "inspect", "--state", p, "--json")
    j = json.loads(out)
    assert rc == 0 and j["node_count"] == 7 and j["accumulated"] == 2 and j["batches_processed"] == 1
    assert {(r["layer"], r["pos"]): r["rank"] for r in j["ranks"]} == rep.ranks()
    bad = bytearray(p.read_bytes())
    bad[0] = ord("Z")
    (tmp_path / "bad.htrs").write_bytes(bytes(bad))
    rc, out = run(cli, "inspect", "--state", tmp_path / "bad.htrs")
    assert rc != 0 and "magic" in out




@pytest.mark.gpu
def test_identical_batches_skip_and_improve_compression(cli, tmp_path):
    rng = np.random.default_rng(271828)
    y = ro.random_tensor([4, 3, 4, 3], rng)
    io.write_batch(y, str(tmp_path / "one.bht"))
    io.write_batch(y, str(tmp_path / "two.bht"))
    rc, out = run(cli, "compress", tmp_path / "one.bht", tmp_path / "two.bht", "--epsilon", "0.25", "--state",
                  tmp_path / "s.htrs", "--stats", tmp_path / "s.csv", "--no-timing")
    assert rc == 0, out
    r = rows(tmp_path / "s.csv")
    assert len(r) == 3 and r[0][2] == "skipped" and r[1][2] == "0" and r[2][2] == "1"
    assert float(r[2][7]) > float(r[1][7])


@pytest.mark.gpu
def test_rte_stabilises_once_the_stream_saturates(cli, tmp_path):
    rng = np.random.default_rng(314)
    bases = [ro.random_orthonormal(5, 2, rng) for _ in range(3)]
    inputs = []
    for k in range(6):
        p = tmp_path / f"b{k}.bht"
        io.write_batch(ro.tucker_family_batch(bases, 2, rng), str(p))
        inputs.append(p)
    (tmp_path / "test").mkdir()
    io.write_batch(ro.tucker_family_batch(bases, 3, rng), str(tmp_path / "test" / "t.bht"))
    rc, out = run(cli, "compress", *inputs, "--epsilon", "0.01", "--state", tmp_path / "s.htrs", "--stats",
                  tmp_path / "s.csv", "--test-dir", tmp_path / "test", "--rte-every", "1", "--no-timing")
    assert rc == 0, out
    r = rows(tmp_path / "s.csv")
    assert len(r) == 7
    prev, skipping = float(r[1][10]), False
    for row in r[2:]:
        rte = float(row[10])
        skipping |= row[2] == "1"
        if skipping:
            assert rte <= prev + 1e-12
        prev = rte
    assert skipping


@pytest.mark.gpu
def test_lock_resume_tolerance_and_shape_drift(cli, tmp_path):
    rng = np.random.default_rng(5)
    io.write_batch(ro.random_tensor([3, 3, 2], rng), str(tmp_path / "a.bht"))
    io.write_batch(ro.random_tensor([3, 3, 2], rng), str(tmp_path / "b.bht"))
    io.write_batch(ro.random_tensor([3, 4, 2], rng), str(tmp_path / "c.bht"))
    (tmp_path / "s.htrs.lock").write_text("\n")
    rc, out = run(cli, "compress", tmp_path / "a.bht", "--epsilon", "0.2", "--state", tmp_path / "s.htrs")
    assert rc != 0 and "lock" in out
    os.remove(tmp_path / "s.htrs.lock")
    assert run(cli, "compress", tmp_path / "a.bht", "--epsilon", "0.2", "--state", tmp_path / "s.htrs")[0] == 0
    assert not (tmp_path / "s.htrs.lock").exists()
    rc, out = run(cli, "compress", tmp_path / "a.bht", tmp_path / "b.bht", "--epsilon", "0.3", "--state",
                  tmp_path / "s.htrs")
    assert rc != 0 and "epsilon" in out
    rc, out = run(cli, "compress", tmp_path / "a.bht", tmp_path / "c.bht", "--epsilon", "0.2", "--state",
                  tmp_path / "s.htrs")
    assert rc != 0 and "shape drift" in out
    st = io.read_state(str(tmp_path / "s.htrs"), device=False)
    assert st.batches_processed == 1 and st.rep.accumulated == 2


@pytest.mark.gpu
def test_decode_indices_and_external_latents(cli, tmp_path):
    from paper_2412_16544_b200 import htrise as ht

    rng = np.random.default_rng(77)
    y = ro.random_tensor([3, 4, 3, 3], rng)
    io.write_batch(y, str(tmp_path / "a.bht"))
    assert run(cli, "compress", tmp_path / "a.bht", "--epsilon", "0.15", "--state", tmp_path / "s.htrs")[0] == 0
    assert run(cli, "decode", "--state", tmp_path / "s.htrs", "--indices", ",", "--out", tmp_path / "none.bht")[0] == 0
    assert not (tmp_path / "none.bht").exists()
    assert run(cli, "decode", "--state", tmp_path / "s.htrs", "--indices", "9", "--out", tmp_path / "x.bht")[0] != 0
    rep = io.read_state(str(tmp_path / "s.htrs")).rep
    lat, _ = ht.encode(rep, y)
    io.write_batch(lat, str(tmp_path / "latent.bht"))
    rc, out = run(cli, "decode", "--state", tmp_path / "s.htrs", "--latent-file", tmp_path / "latent.bht", "--out",
                  tmp_path / "full.bht")
    assert rc == 0, out
    assert np.array_equal(io.read_batch(str(tmp_path / "full.bht")), ht.decode(rep, lat))
    rc, out = run(cli, "decode", "--state", tmp_path / "s.htrs", "--indices", "1-2", "--out", tmp_path / "two.bht")
    assert rc == 0, out
    two = io.read_batch(str(tmp_path / "two.bht"))
    for m in range(2):
        assert np.linalg.norm(two[..., m] - y[..., m]) <= (0.15 + 1e-9) * np.linalg.norm(y)


@pytest.mark.gpu
def test_acceptance_c9_resume_is_byte_identical(cli, tmp_path):
    """acceptance.cpp:401-507: an interrupted-and-resumed run equals the
    uninterrupted one byte for byte (state and stats CSV); permuted
    containers with --permute give the same stats; decoded slices honour the
    recorded normalisation."""
    rng = np.random.default_rng(999999)
    inputs = []
    for k in range(7):
        p = tmp_path / f"b{k}.bht"
        io.write_batch(ro.random_tensor([4, 3, 4, 2], rng), str(p))
        inputs.append(p)
    common = ["--epsilon", "0.2", "--normalize", "maxabs", "--no-timing"]
    assert run(cli, "compress", *inputs, *common, "--state", tmp_path / "a.htrs", "--stats", tmp_path / "a.csv")[0] == 0
    assert run(cli, "compress", *inputs[:3], *common, "--state", tmp_path / "b.htrs", "--stats",
               tmp_path / "b.csv")[0] == 0
    assert run(cli, "compress", *inputs, *common, "--state", tmp_path / "b.htrs", "--stats", tmp_path / "b.csv")[0] == 0
    assert (tmp_path / "a.htrs").read_bytes() == (tmp_path / "b.htrs").read_bytes()
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
    permuted = []
    for k, p in enumerate(inputs):
        b = io.read_batch(str(p))
        q = tmp_path / f"p{k}.bht"
        io.write_batch(np.transpose(b, (3, 1, 0, 2)), str(q))  # batch first
        permuted.append(q)
    assert run(cli, "compress", *permuted, *common, "--permute", "2,1,3,0", "--state", tmp_path / "c.htrs", "--stats",
               tmp_path / "c.csv")[0] == 0
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "c.csv").read_bytes()
    st = io.read_state(str(tmp_path / "a.htrs"), device=False)
    io.write_state(st, str(tmp_path / "again.htrs"))
    assert (tmp_path / "a.htrs").read_bytes() == (tmp_path / "again.htrs").read_bytes()
    assert run(cli, "decode", "--state", tmp_path / "a.htrs", "--indices", "1-2", "--out", tmp_path / "dec.bht")[0] == 0
    dec = io.read_batch(str(tmp_path / "dec.bht"))
    want = io.read_batch(str(inputs[0]))[..., 0:2]
    assert np.linalg.norm(dec - want) / np.linalg.norm(want) <= 0.2 + 1e-9
