"""The C++ drop-in boundary: include/htrise/*.hpp (reference API names and
semantics) compile standalone, and a reference-style test program written
against them passes on the GPU through libhtrise_cuda.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = ["tensor.hpp", "dimension_tree.hpp", "truncated_svd.hpp", "bht.hpp", "ht_rise.hpp", "metrics.hpp",
           "htrise.hpp", "device.hpp", "json.hpp", "io.hpp"]


@pytest.mark.parametrize("header", HEADERS)
def test_header_compiles_standalone(header, tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(f'#include <htrise/{header}>\nint main() {{ return 0; }}\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", str(src)], check=True)


def test_c_header_is_plain_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include <htrise_cuda.h>\nint main(void) { htr_node n; (void)n; return 0; }\n')
    subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src)], check=True)


@pytest.mark.gpu
def test_dropin_program_passes_on_gpu():
    from paper_2412_16544_b200 import build

    binary = build.DROPIN_BIN
    if not os.path.exists(binary):
        build.build_dropin_test()
    r = subprocess.run([binary], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0 and "ALL PASSED" in r.stdout
