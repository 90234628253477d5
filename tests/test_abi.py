"""CPU-side checks of the boundary: libgcp.so loads, exports every symbol the
header declares, and the pure host entry points behave (no GPU needed)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _header_symbols():
    text = (ROOT / "include" / "gcp.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:gcp_status|void|const char\*)\s+(gcp_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    import paper_2605_20353_b200 as g
    declared = _header_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(g.lib, name), name
    assert set(declared) == set(g.SYMBOLS)


def test_library_is_sm100a_only():
    import subprocess
    so = ROOT / "paper_2605_20353_b200" / "libgcp.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_grid_plan_host_entry_point(orc):
    import paper_2605_20353_b200 as g
    for dims, P in [((4821207, 1774269, 1805187), 8), ((10000, 10000, 10000), 4), ((300, 200, 100), 12),
                    ((1605, 4198, 1631, 4209, 868131), 8)]:
        grid, lo, hi = g.gcp_grid_plan(P, dims)
        assert grid == orc.grid_plan(P, dims)[0]
        for w in range(P):
            olo, ohi = orc.block_bounds(dims, grid, w)
            assert list(lo[w]) == olo and list(hi[w]) == ohi


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_20353_b200 as g
    with pytest.raises(g.GcpError):
        g.Context(0)
