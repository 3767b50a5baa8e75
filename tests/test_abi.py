"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/reachplan_b200.h declares, mirrors the reference defaults, and
fails loudly (no CPU fallback) when no CUDA device is present."""
import ctypes as C
import os

import pytest

from paper_1906_10678_b200 import abi, api, scenes


def test_library_exports_every_header_symbol():
    L = api.lib()
    names = api.header_symbols()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.rp_abi_version() == 1


def test_struct_layouts_match_header():
    # sizes the C compiler gives the header structs (x86-64)
    assert C.sizeof(abi.Arm) == 4 * 4 + 8 * (4 + 3 + 1 + 16 + 4 + 3 + 1 + 3 + 3)
    assert C.sizeof(abi.Pose) == 4 * 8 + 8 + 8 * 3 * (4 + 5 + 4)
    assert C.sizeof(abi.SolveStats) == 13 * 8 + 8
    assert C.sizeof(abi.Obstacle) == 8 + 6 * 8 + 8 + 8 + 8


def test_defaults_mirror_reference():
    L = api.lib()
    a = abi.Arm()
    L.rp_arm_init(C.byref(a), 4, (C.c_double * 4)(0.5, 0.5, 0.5, 0.125))
    assert tuple(a.base_axis) == (0, 0, 1) and tuple(a.base_ref) == (1, 0, 0)
    assert tuple(a.fold_plane_normal) == (0, 1, 0)
    assert abs(a.fold_flex - abi.deg2rad(170.0)) < 1e-15
    r = abi.ReachParams()
    L.rp_reach_params_init(C.byref(r))
    assert (r.n_samples, r.mode, r.epsilon_gap, r.near_target_radius) == (8, 1, -1.0, -1.0)
    p = abi.PathParams()
    L.rp_path_params_init(C.byref(p))
    assert list(p.relax_schedule[:p.n_relax]) == [1.5, 2.0, 3.0] and p.unfold_steps == 16
    # derived parameters of the synthetic arm
    arm, rp = scenes.config("C2").arm(), scenes.config("C2").reach_params()
    assert L.rp_nominal_spacing(C.byref(arm), C.byref(rp)) == 0.0625
    assert L.rp_resolved_epsilon(C.byref(arm), C.byref(rp)) == 0.03125
    assert L.rp_resolved_near_radius(C.byref(arm), C.byref(rp)) == 0.03125
    assert L.rp_effective_dilation(C.byref(arm), C.byref(rp), -1.0) == 0.098125


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    with pytest.raises(api.ReachplanError) as e:
        api.Context(0)
    assert e.value.code == abi.RP_E_CUDA


def test_header_has_no_torch_types():
    hdr = open(os.path.join(os.path.dirname(api.HERE), "include", "reachplan_b200.h")).read()
    assert "torch" not in hdr.lower().replace("no torch", "")
    assert 'extern "C"' in hdr
