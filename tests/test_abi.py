"""The C-ABI library without a GPU: it loads, exports every symbol
include/uniap.h declares, and its host-only entry points (Algorithm 1's
candidate list, the strategy catalogue, the record pick) behave (CPU only)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2307_16375_b200 as pkg
from paper_2307_16375_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "uniap.h")).read()
    return sorted(set(re.findall(r"\b(uniap_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(pkg.LIB_PATH), "run python build.py"
    out = subprocess.run(["nm", "-D", "--defined-only", pkg.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(uniap_\w+)", out))
    declared = _declared()
    assert declared and set(declared) <= exported, set(declared) - exported
    lib = pkg.lib()
    for name in declared:
        assert hasattr(lib, name)
    assert set(binding.EXPORTS) == set(declared)


def test_library_targets_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_k2_uses_dpx_viaddmnmx():
    """The chain DP's min-plus relaxation is one DPX VIADDMNMX on sm_100a."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun",
                          "_ZN5uniap8k2_chainILi10ELi8ELi512ELb0ELb0ELb0EEEvNS_6K2ArgsE", pkg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert out.count("VIADDMNMX") >= 50


def test_every_planned_kernel_shape_is_compiled():
    rc, case = pkg.selftest()
    assert rc == 0, f"no kernel for (S, Q, single) = {case}"


def test_record_layout():
    assert pkg.RECORD_BYTES == C.sizeof(binding.uniap_record) == 8 + 6 * 4 + 2 * 64 * 4 + 2 * 64 * 8 + 64 * 4 + 24


def test_candidates_and_catalogue_match_the_oracle(orc):
    for n in (1, 2, 4, 6, 8, 12, 16, 32):
        for B in (1, 2, 6, 8, 32, 64, 128):
            assert pkg.candidates(n, B) == orc.candidates(n, B)
    for g in (1, 2, 3, 4, 6, 8, 12, 16, 32):
        for space in (0, 1):
            assert pkg.catalogue(g, space) == orc.catalogue(g, space)
    assert len(pkg.candidates(8, 32)) == 16 and len(pkg.candidates(4, 6)) == 7


def _rec(obj, deg, c, cfg, L=4):
    r = binding.uniap_record()
    r.objective, r.deg, r.c, r.cfg_index, r.L = obj, deg, c, cfg, L
    for u in range(L):
        r.stage_of[u] = u * deg // L
        r.strategy_of[u] = cfg
    r.dp_cells, r.dp_relax, r.dp_cells_canonical = 10, 20, 30
    return bytes(r)


def test_pick_orders_by_objective_then_deg_then_c():
    recs = _rec(7, 2, 4, 5) + _rec(7, 2, 2, 4) + _rec(9, 1, 1, 0) + _rec(pkg.INT64_MAX, 0, 0, -1)
    st, r = pkg.pick(recs, 4)
    assert st == 0 and (r["objective"], r["deg"], r["c"], r["cfg_index"]) == (7, 2, 2, 4)
    assert r["dp_cells"] == 40 and r["dp_relax"] == 80 and r["dp_cells_canonical"] == 120
    st, r = pkg.pick(_rec(pkg.INT64_MAX, 0, 0, -1) * 2, 2)
    assert st == binding.UNIAP_ERR_INFEASIBLE and r["objective"] == pkg.INT64_MAX


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.UniapError):
        pkg.Handle(0)
