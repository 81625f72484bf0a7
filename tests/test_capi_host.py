"""CPU tests: the C-ABI library loads and exports every declared symbol, and
the host-side mirror of the reference interface validates like the
reference (no GPU needed, no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fpmimo_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2504_09820_b200 import build
    build.build()
    from paper_2504_09820_b200 import _lib
    return _lib.load()


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fpm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    from paper_2504_09820_b200 import _lib
    assert set(_declared()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(os.path.join(ROOT, "paper_2504_09820_b200", "libfpmimo_b200.so"))
    for name in _declared():
        assert hasattr(raw, name), name


def test_no_gpu_calls_work(lib):
    assert lib.fpm_version() >= 10000
    assert lib.fpm_strerror(2).decode() == "non-PD diagonal block"
    n, l_, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.fpm_limits(ctypes.byref(n), ctypes.byref(l_), ctypes.byref(m)) == 0
    assert n.value >= 128 and l_.value >= 8 and m.value >= 512


def test_argument_validation_without_gpu(lib):
    from paper_2504_09820_b200 import _lib
    ps = _lib.Precision(_lib.Format(53, 11, 1), _lib.Format(11, 5, 1), _lib.Format(11, 5, 1))
    dummy = ctypes.c_void_p(16)
    # iters < 1, bad rho variant, work coarser than matvec: all rejected before any CUDA call
    assert lib.fpm_cg(dummy, dummy, None, 1, 8, 1, 0, ps, 0, dummy, dummy, dummy, None) == 1
    assert lib.fpm_cg(dummy, dummy, None, 1, 8, 1, 3, ps, 7, dummy, dummy, dummy, None) == 1
    bad = _lib.Precision(_lib.Format(11, 5, 1), _lib.Format(53, 11, 1), _lib.Format(53, 11, 1))
    assert lib.fpm_cg(dummy, dummy, None, 1, 8, 1, 3, bad, 0, dummy, dummy, dummy, None) == 1
    # device complex128 arrays off 16-byte alignment: rejected before any launch
    odd = ctypes.c_void_p(24)
    assert lib.fpm_cg(odd, dummy, None, 1, 8, 1, 3, ps, 0, dummy, dummy, dummy, None) == 1
    assert lib.fpm_cg(dummy, dummy, None, 1, 8, 1, 3, ps, 0, odd, dummy, dummy, None) == 1
    assert lib.fpm_gram(odd, dummy, 1, 16, 8, 0.1, dummy, dummy, None) == 1
    assert lib.fpm_lmmse(dummy, odd, 1, 8, dummy, None, None) == 1
    assert lib.fpm_detect(dummy, odd, None, 1, 16, 8, 0.1, 3, 4, 4, ps, 0, 16, None, dummy, dummy, dummy,
                          None, dummy, None) == 1
    # L must divide N for the detector (build_blocks_batch default)
    assert lib.fpm_detect(dummy, dummy, None, 1, 16, 8, 0.1, 3, 3, 4, ps, 0, 16, None, dummy, dummy, dummy,
                          None, dummy, None) == 1
    assert lib.fpm_slice_count(dummy, None, 1, 4, 32, None, dummy, None) == 1
    assert lib.fpm_bj_setup(dummy, 1, 8, 3, 0, dummy, None, None) == 1
    # convergence-study diagnostics (csrc/fpm_diag.cu): empty batches are no-ops,
    # misaligned / missing arrays and N > 128 are rejected before any launch
    assert lib.fpm_herm_norm2(None, 0, 8, None, None) == 0
    assert lib.fpm_herm_norm2(dummy, 1, 8, None, None) == 1
    assert lib.fpm_herm_norm2(odd, 1, 8, dummy, None) == 1
    assert lib.fpm_herm_norm2(dummy, 1, 129, dummy, None) == _lib.FPM_EUNSUPPORTED
    assert lib.fpm_residual_gaps(None, None, None, None, None, 0, 8, 4, None, None) == 0
    assert lib.fpm_residual_gaps(dummy, dummy, dummy, dummy, dummy, 1, 8, 0, dummy, None) == 0
    assert lib.fpm_residual_gaps(dummy, dummy, dummy, None, dummy, 1, 8, 4, dummy, None) == 1
    assert lib.fpm_residual_gaps(dummy, odd, dummy, dummy, dummy, 1, 8, 4, dummy, None) == 1
    assert lib.fpm_residual_gaps(dummy, dummy, dummy, dummy, dummy, 1, 129, 4, dummy, None) == _lib.FPM_EUNSUPPORTED


def test_detector_spec_mirrors_reference_validation():
    from paper_2504_09820_b200.detect import DetectorSpec
    from paper_2504_09820_b200.errors import ContractViolation
    with pytest.raises(ContractViolation):
        DetectorSpec(algorithm="fp_bj_cg")
    with pytest.raises(ContractViolation):
        DetectorSpec(algorithm="zf_direct")
    d = DetectorSpec(algorithm="fp_cg", matvec="fp16", inner="fp16")
    assert d.name == "fp_cg[fp16]"
    assert d.precision().labels() == ("fp64", "fp16", "fp16")
    assert DetectorSpec("cg", matvec="fp16").precision().is_native


def test_precision_config_rules():
    from paper_2504_09820_b200.errors import ContractViolation, FormatError
    from paper_2504_09820_b200.formats import FP16, FP64, make_format
    from paper_2504_09820_b200.solvers import PrecisionConfig
    with pytest.raises(ContractViolation):
        PrecisionConfig(work=FP16, matvec=FP64, inner=FP64)
    assert PrecisionConfig.uniform(FP16).labels() == ("fp16", "fp16", "fp16")
    with pytest.raises(FormatError):
        make_format(60, 11)
    assert make_format(11, 5).triple() == (11, 5, 1)


def test_block_packing_round_trip():
    from paper_2504_09820_b200.solvers import BatchBlocks, pack_blocks
    rng = np.random.default_rng(0)
    mats = [rng.standard_normal((3, 3, 3)) + 0j, rng.standard_normal((3, 3, 3)) + 0j,
            rng.standard_normal((3, 2, 2)) + 0j]
    packed = pack_blocks(mats, 8, 3)
    back = BatchBlocks(packed, 8, 3).mats
    for a, b in zip(mats, back):
        np.testing.assert_array_equal(a, b)


def test_format_registry_matches_reference_names():
    from paper_2504_09820_b200.formats import registered_formats
    reg = registered_formats()
    assert {k: v.triple() for k, v in reg.items()} == {
        "bfloat16": (8, 8, 1), "fp16": (11, 5, 1), "fp32": (24, 8, 1), "fp64": (53, 11, 1)}


def test_product_library_has_no_trace_state(lib):
    """Diagnostics are compile-time only (-DFPM_DIAG): the product library
    refuses a trace buffer instead of keeping global state."""
    from paper_2504_09820_b200 import _lib
    assert lib.fpm_debug_set_trace(ctypes.c_void_p(256)) == _lib.FPM_EUNSUPPORTED
    assert lib.fpm_debug_set_trace(None) == _lib.FPM_EUNSUPPORTED


def test_no_per_call_getenv_in_library_sources():
    """Planner knobs come from the load-time snapshot (fpm_host.cu knob()),
    never from a per-call getenv."""
    import glob
    srcs = glob.glob(os.path.join(ROOT, "paper_2504_09820_b200", "csrc", "*.cu*"))
    hits = [(p, i) for p in srcs for i, line in enumerate(open(p), 1) if "getenv(" in line]
    assert not hits, hits


def test_build_stamp_tracks_flags(monkeypatch):
    """The build stamp covers the nvcc flags, so a prebuilt library compiled
    with other flags (or from other sources) is rebuilt, not reused."""
    from paper_2504_09820_b200 import build as B
    B.build()
    assert not B.needs_build()
    s0 = B._stamp()
    monkeypatch.setattr(B, "FLAGS", B.FLAGS + ["-DFPM_SOMETHING_ELSE"])
    assert B._stamp() != s0 and B.needs_build()


def test_format_extremes_match_reference_definition():
    """FloatFormat.x_min / x_max (formats.py:60-61, 83-88)."""
    from paper_2504_09820_b200.formats import BFLOAT16, FP16, FP32, FP64, make_format
    assert FP16.x_max == 65504.0 and FP16.x_min == 2.0 ** -14
    assert BFLOAT16.x_max == float.fromhex("0x1.fep+127") and BFLOAT16.x_min == 2.0 ** -126
    assert FP32.x_max == float.fromhex("0x1.fffffep+127") and FP32.x_min == 2.0 ** -126
    assert FP64.x_max == float.fromhex("0x1.fffffffffffffp+1023") and FP64.x_min == 2.0 ** -1022
    f = make_format(5, 4)
    assert f.x_max == (2 - 2 ** -4) * 2 ** 7 and f.x_min == 2.0 ** -6
