"""The C-ABI library loads and exports every symbol include/ermc_b200.h
declares (no compute calls: this runs on the CPU container)."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

from paper_1810_00188_b200 import capi

HEADER = Path(__file__).resolve().parent.parent / "include" / "ermc_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ermc_b200_\w+)\s*\(", text)))


def test_header_declares_boundary():
    names = declared()
    for must in ("ermc_b200_solve", "ermc_b200_solve_range", "ermc_b200_session_create",
                 "ermc_b200_session_solve", "ermc_b200_trace_rays"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(capi.EXPORTS) == set(declared())


def test_abi_version_and_defaults():
    lib = capi.load()
    assert lib.ermc_b200_abi_version() == 2
    c = capi.Config()
    lib.ermc_b200_config_default(ctypes.byref(c))
    assert (c.rays_per_cell, c.tolerance, c.max_steps, c.steps_per_level, c.coarsen_ratio) == \
        (2000, 1e-4, 100000, 5, 2)
    assert c.precision == capi.FP64 and c.device == -1 and c.n_devices == 1
    assert capi.default_config_values()["n_devices"] == 1


def test_struct_layouts_match_header(tmp_path):
    # sizeof/offsetof from the C compiler vs the ctypes mirror.
    import subprocess
    fields = {"ermc_grid_t": (capi.Grid, ["nx", "dx", "origin"]),
              "ermc_boundary_t": (capi.Boundary, ["kind", "lo_temperature", "hi_emissivity"]),
              "ermc_model_t": (capi.Model, ["n_bands", "band_nu_lo", "ib_table"]),
              "ermc_config_t": (capi.Config, ["rays_per_cell", "tolerance", "seed", "max_steps",
                                              "sorting", "precision", "device"]),
              "ermc_solution_t": (capi.Solution, ["q_r", "total_steps", "wall_time"]),
              "ermc_ray_result_t": (capi.RayResult, ["q_contribution", "dir", "steps",
                                                     "next_draw"]),
              "ermc_ray_state_t": (capi.RayState, ["pos", "cell", "transmissivity", "band",
                                                   "prefactor", "reflections", "seed",
                                                   "cell_id", "ray_id", "next_draw"])}
    src = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(){"]
    for t, (_, fs) in fields.items():
        src.append(f'printf("{t} %zu\\n", sizeof({t}));')
        for f in fs:
            src.append(f'printf("{t}.{f} %zu\\n", offsetof({t}, {f}));')
    src.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    got = dict(line.split() for line in out.splitlines())
    for t, (cls, fs) in fields.items():
        assert int(got[t]) == ctypes.sizeof(cls), t
        for f in fs:
            assert int(got[f"{t}.{f}"]) == getattr(cls, f).offset, (t, f)
