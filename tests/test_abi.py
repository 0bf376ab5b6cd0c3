"""CPU-side checks of the C-ABI boundary (-m "not gpu"): the library builds/loads, exports
every symbol include/ssi.h declares, and its synchronous validation and workspace
queries work without a GPU (no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ssi.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"SSI_API\s+[\w\s\*]+?\b(ssi_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2411_05510_b200 import build, _lib
    build.build()
    return _lib.get()


def test_header_declares_the_five_entry_points():
    names = _declared()
    for n in ("ssi_covariances", "ssi_toeplitz", "ssi_rsvd", "ssi_modal_sweep", "ssi_stab3d"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_python_binding_covers_every_symbol():
    from paper_2411_05510_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_status_strings_and_version(lib):
    assert lib.ssi_status_string(0) == b"ok"
    assert b"workspace" in lib.ssi_status_string(4)
    assert b"sm_100a" in lib.ssi_version()


def test_workspace_queries_are_host_only(lib):
    b = C.c_size_t(0)
    assert lib.ssi_covariances_ws(360000, 192, 1, 119, 0, C.byref(b)) == 0 and b.value > 0
    assert lib.ssi_rsvd_ws(11520, 220, 200, C.byref(b)) == 0 and b.value > 11520 * 220 * 8 * 4
    assert lib.ssi_modal_sweep_ws(192, 60, 2, 200, 2, C.byref(b)) == 0 and b.value > 0


def test_synchronous_validation_without_gpu(lib):
    """Argument errors are reported before any launch (no device needed)."""
    b = C.c_size_t(0)
    assert lib.ssi_rsvd_ws(100, 0, 1, C.byref(b)) == 1              # k < 1
    assert lib.ssi_rsvd_ws(100, 20, 30, C.byref(b)) == 1            # n_keep > k
    assert lib.ssi_modal_sweep_ws(6, 20, 3, 30, 2, C.byref(b)) == 1   # odd order
    assert lib.ssi_covariances_ws(100, 6, 1, 9, 7, C.byref(b)) == 3   # unknown mode
    dummy = C.c_void_p(16)
    # record too short: lag_hi >= N
    assert lib.ssi_covariances(dummy, 0, 10, 6, 6, 1, 10, 0, 0, 10, 1, dummy, dummy, 1 << 20, None) == 1
    assert b"too short" in lib.ssi_last_error()
    # ldY < l
    assert lib.ssi_covariances(dummy, 0, 100, 6, 5, 1, 9, 0, 0, 100, 1, dummy, dummy, 1 << 20, None) == 2
    # workspace too small
    assert lib.ssi_covariances(dummy, 0, 100, 6, 6, 1, 9, 0, 0, 100, 1, dummy, dummy, 8, None) == 4
    # toeplitz ld
    assert lib.ssi_toeplitz(dummy, 6, 20, dummy, 100, None) == 2
    # rsvd: n_keep > k
    assert lib.ssi_rsvd(dummy, 120, 120, 40, 2, 1, 1, 41, dummy, 120, dummy, dummy, 1 << 30, None) == 1


def test_oracle_is_not_imported_by_the_product():
    """The product package never imports the oracle (independence)."""
    pkg = os.path.join(ROOT, "paper_2411_05510_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace("no oracle", ""), f


def test_oracle_is_not_imported_by_the_tools():
    """Only tests/, smoke() and bench.py's CPU legs may execute the oracle: the measurement scripts
    under tools/ take their presets from the product (api.CRITERIA_*); scripts that compare with the
    oracle live under tests/tools/."""
    for f in sorted(os.listdir(os.path.join(ROOT, "tools"))):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "tools", f)).read()
            assert not re.search(r"^\s*(import|from)\s+.*\boracle\b", txt, re.M), f


def test_rsvd_workspace_is_monotone_in_m(lib):
    """A workspace sized for the largest lag of a sweep (c4: i = 20..80) serves every lag."""
    b = C.c_size_t(0)
    prev = 0
    for i in range(20, 81):
        assert lib.ssi_rsvd_ws(192 * i, 220, 200, C.byref(b)) == 0
        assert b.value >= prev, i
        prev = b.value


def test_rsvd_toeplitz_workspace_and_validation(lib):
    """Structured RSVD: workspace non-decreasing in i (one workspace serves a lag sweep);
    argument errors before any launch."""
    b = C.c_size_t(0)
    prev = 0
    for i in range(20, 81, 4):
        assert lib.ssi_rsvd_toeplitz_ws(192, i, 220, 200, C.byref(b)) == 0
        assert b.value >= prev, i
        prev = b.value
    assert lib.ssi_rsvd_toeplitz_ws(6, 2, 13, 1, C.byref(b)) == 1      # k > l*i
    dummy = C.c_void_p(16)
    assert lib.ssi_rsvd_toeplitz(dummy, 6, 20, 40, 2, 1, 1, 41, dummy, 120, dummy, dummy, 1 << 30, None) == 1
    assert lib.ssi_rsvd_toeplitz(dummy, 6, 20, 40, 2, 1, 1, 30, dummy, 119, dummy, dummy, 1 << 30, None) == 2
    assert lib.ssi_rsvd_toeplitz(dummy, 6, 20, 40, 2, 1, 1, 30, dummy, 120, dummy, dummy, 64, None) == 4


def test_spectral_covariance_workspace_and_validation(lib):
    """SSI_COV_SPECTRAL (= 2): host-side plan / workspace query, lag limit, shard monotonicity."""
    b = C.c_size_t(0)
    assert lib.ssi_covariances_ws(360000, 192, 1, 119, 2, C.byref(b)) == 0
    full = b.value
    # segment spectra of the c3 record: X and Ye, each (F/2+1) x 2S x lp doubles (F = 1024, S = 398)
    assert full >= 513 * 2 * 398 * 2 * 192 * 8
    assert lib.ssi_covariances_ws(360000, 192, 1, 2048, 2, C.byref(b)) == 3     # lag_hi >= 2048
    F, S = C.c_int32(0), C.c_int64(0)
    assert lib.ssi_cov_spectral_plan(360000, 192, 1, 119, C.byref(F), C.byref(S)) == 0
    assert (F.value, S.value) == (1024, 398)          # flop model minimum at c3
    assert lib.ssi_cov_spectral_plan(360000, 192, 1, 159, C.byref(F), C.byref(S)) == 0
    assert F.value > 159 and S.value == -(-360000 // (F.value - 159))
    assert lib.ssi_covariances_ws(6000, 7, 1, 39, 2, C.byref(b)) == 0 and b.value > 0   # odd l
    dummy = C.c_void_p(16)
    assert lib.ssi_covariances(dummy, 0, 360000, 192, 192, 1, 119, 2, 0, 360000, 1, dummy, dummy, 8, None) == 4
    # segments are processed in chunks: a day-long record needs no more spectra workspace
    assert lib.ssi_covariances_ws(8_640_000, 192, 1, 119, 2, C.byref(b)) == 0
    assert b.value < 4 * full


def test_int8x3_channel_counts_rejected_synchronously(lib):
    """SSI_COV_INT8X3 (= 1) tiles channels by 64 (or one tile of 16..64): any other l is rejected
    by the workspace query and by ssi_covariances with SSI_ERR_DTYPE (= 3), before any work —
    the query used to divide by a zero tile width (SIGFPE) for l = 6."""
    b = C.c_size_t(0)
    for l in (6, 7, 33, 72, 100):
        assert lib.ssi_covariances_ws(6000, l, 1, 39, 1, C.byref(b)) == 3, l
    for l in (16, 48, 64, 192, 256):
        assert lib.ssi_covariances_ws(6000, l, 1, 39, 1, C.byref(b)) == 0 and b.value > 0, l
    dummy = C.c_void_p(16)
    assert lib.ssi_covariances(dummy, 0, 6000, 6, 6, 1, 39, 1, 0, 6000, 1, dummy, dummy, 1 << 30, None) == 3
