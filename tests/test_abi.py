"""The C ABI library: loads, exports every symbol include/fxg.h declares, and its
pure host entry points (profiles, groups, columns, synthetic generators) match
the reference.  No device compute here (CPU-only container)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2603_12016_b200 as fx
from paper_2603_12016_b200 import fxg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fxg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(fx_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = fxg.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.fx_abi_version() == 1


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {fxg.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_profiles_and_errors():
    p = fx.resolve_profile("performance")
    assert p.ng == 32 and p.n_angles == 1 and p.symmetric == 0
    p = fx.resolve_profile("ibsi-like")
    assert p.ng == 256 and p.n_angles == 4 and p.symmetric == 1
    with pytest.raises(fx.FxError) as e:
        fx.resolve_profile("bogus")
    assert e.value.kind == "UnknownProfile"


def test_group_resolution_canonical_order():
    assert fx.resolve_groups(["*ALL*"]) == 0x7F
    assert fx.resolve_groups(["shape", "intensity"]) == 0x03
    for bad in (["intensity", "nope"], []):
        with pytest.raises(fx.FxError) as e:
            fx.resolve_groups(bad)
        assert e.value.kind == "ConfigError"


@pytest.mark.parametrize("profile", ["default", "performance", "ibsi-like"])
def test_columns_match_reference(reference, profile):
    from oracle import make_params
    for groups in (["intensity"], ["moments"], ["glcm"], ["*ALL*"], ["glrlm", "ngtdm"]):
        assert fx.feature_columns(groups, fx.resolve_profile(profile)) == \
            reference.columns(groups, make_params(profile))


def test_column_counts():
    counts = {"default": 427, "performance": 292, "ibsi-like": 427}
    for prof, n in counts.items():
        assert len(fx.feature_columns(["*ALL*"], fx.resolve_profile(prof))) == n
    cols = fx.feature_columns(["glcm"], fx.resolve_profile("performance"))
    assert cols[:2] == ["glcm_asm_0", "glcm_asm_ave"]


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(fx.FxError) as e:
        fx.Context(0)
    assert e.value.kind == "CudaError"


def test_unsupported_groups_have_no_cpu_fallback():
    """shape/glrlm/glszm/ngtdm have no device kernel yet: ConfigError, never CPU."""
    lib = fxg.lib()
    p = fx.resolve_profile("default")
    h = ctypes.c_void_p()
    rc = lib.fx_roi_features(None, None, None, None, ctypes.c_size_t(0), ctypes.c_uint(2),
                             ctypes.byref(p), None, ctypes.c_size_t(0))
    assert rc == 11  # FX_E_ARG: no ctx -> never computes on the host
    del h
