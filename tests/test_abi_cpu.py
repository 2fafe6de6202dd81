"""C-ABI checks that need no GPU: the in-tree library loads, exports every
function include/mars_b200.h declares, and the ctypes struct layouts match
the C layouts (verified with gcc against the header)."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_2604_26963_b200 import _native as N
from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mars_b200.h")


def _declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(mars_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        import __graft_entry__ as g

        g.build()
    return N.load()


def test_library_exports_every_declared_symbol(lib):
    declared = _declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(N.EXPORTS)


def test_abi_version(lib):
    assert lib.mars_abi_version() == 7


def test_default_config_matches_reference_constants(lib):
    cfg = N.MarsConfig()
    lib.mars_config_default(ctypes.byref(cfg))
    assert (cfg.block_size, cfg.token_budget, cfg.tick_duration_s) == (16, 512, 0.064)
    assert list(cfg.level_bounds)[:3] == [4000, 32000, 128000]
    assert list(cfg.level_quotas)[:3] == [2000, 8000, 32000]
    assert (cfg.window_size, cfg.max_decode_slots, cfg.max_promotions) == (128, 64, 3)
    assert (cfg.promotion_wait_s, cfg.deadline_slack, cfg.max_pin_horizon_s) == (10.0, 2.0, 60.0)
    assert (cfg.w_min, cfg.initial_window, cfg.reserve_fraction) == (2, 8.0, 0.10)
    assert (cfg.kv_high_watermark, cfg.kv_low_watermark, cfg.hysteresis_window) == (0.9, 0.7, 3)


def test_create_without_gpu_fails_loudly(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = N.MarsConfig()
    lib.mars_config_default(ctypes.byref(cfg))
    ctx = ctypes.c_void_p()
    rc = lib.mars_create(ctypes.byref(cfg), 0, 16, 16, ctypes.byref(ctx))
    assert rc == N.MARS_ERR_CUDA


STRUCTS = {
    "mars_config": N.MarsConfig, "mars_cols": N.MarsCols, "mars_scalars": N.MarsScalars,
    "mars_step_in": N.MarsStepIn, "mars_step_out": N.MarsStepOut,
    "mars_kv_config": N.MarsKvConfig,
}


def test_ctypes_layouts_match_the_c_header():
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(){"]
    for cname, py in STRUCTS.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-o", exe, src], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = dict(l.split() for l in out.strip().splitlines())
    for cname, py in STRUCTS.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"
