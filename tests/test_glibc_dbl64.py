"""CPU: csrc/glibc_dbl64.cuh (kernel (1)'s sin/cos/asin) equals the libm the
reference links against, bit for bit.

The header is compiled for the host (g++, -ffp-contract=off so only its
explicit fma() calls fuse) and checked against libm's own sin/cos/asin on
random arguments in every branch range of glibc's s_sin.c / e_asin.c, +-64
ulp around every branch boundary, the special values, and the haversine's
own argument distributions (tests/native/glibc_dbl64_check.cpp). The device
build of the same header is checked by the GPU tests' bit-identical tables.
"""
import subprocess
from pathlib import Path

import pytest

from paper_2001_05291_b200 import _glibc_tables

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_2001_05291_b200" / "csrc"


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    _glibc_tables.write()
    exe = tmp_path_factory.mktemp("gl") / "glibc_dbl64_check"
    subprocess.run(["g++", "-O2", "-mfma", "-ffp-contract=off", "-std=c++17", f"-I{CSRC}",
                    str(ROOT / "tests" / "native" / "glibc_dbl64_check.cpp"), "-o", str(exe),
                    "-lm"], check=True)
    return exe


@pytest.mark.parametrize("seed", [1, 2])
def test_sin_cos_asin_bit_identical_to_libm(checker, seed):
    r = subprocess.run([str(checker), "300000", str(seed)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:]
    assert r.stdout.strip().endswith("0 mismatches"), r.stdout[-2000:]


def test_tables_come_from_the_pinned_libm():
    tabs = _glibc_tables.extract()
    assert [len(v) for v in tabs.values()] == [n for _, _, n in _glibc_tables.TABLES]
    # __sincostab row 0 is (sin 0, 0, cos 0, 0); powtwo holds 2^i
    assert tabs["kSinCosTab"][:4] == [0.0, 0.0, 1.0, 0.0]
    assert tabs["kPowTwo"][:4] == [1.0, 2.0, 4.0, 8.0]
