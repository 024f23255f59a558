"""C-ABI library: loads without a GPU, exports every symbol include/kvf.h
declares, and its host-side validation mirrors the reference's ValueErrors."""

import ctypes

import pytest

from paper_2602_09725_b200 import _lib, layout as L


def test_library_loads_and_exports_declared_symbols():
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert "kvf_restore" in declared and "kvf_pack_frames" in declared
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.kvf_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header_sizes():
    # kvf_plan: 15 x i32; kvf_surface: ptr + 3 x i64; kvf_paged: 3 ptr + ptr + 2 i32 + 3 i64 + 2 i32
    assert ctypes.sizeof(_lib.kvf_plan) == 60
    assert ctypes.sizeof(_lib.kvf_surface) == 32
    assert ctypes.sizeof(_lib.kvf_paged) == 72


@pytest.mark.parametrize("res", L.RESOLUTION_ORDER)
@pytest.mark.parametrize("T", [1, 5, 1000, 10000])
def test_plan_init_matches_host_plan(res, T):
    for cfg in L.tiling_candidates(8, 128)[::5]:
        plan = L.plan_inter_frame(T, res, cfg, 4)
        c = plan.to_c(128)
        assert (c.frame_h, c.frame_w, c.frame_count) == (plan.frame_h, plan.frame_w,
                                                        plan.frame_count)
        assert _lib.load().kvf_plan_frame_bytes(c) == plan.frame_count * 3 * plan.frame_h * plan.frame_w


def test_plan_validation_raises_value_error():
    p = _lib.kvf_plan(10, 12, 64, 3, 4, 8, 8, 4, 16, 4, 4, 0, 0, 0, 8)
    with pytest.raises(ValueError, match="powers of two"):
        _lib.call("kvf_plan_init", p)
    p = _lib.kvf_plan(10, 8, 128, 1, 8, 1, 128, 4, 16, 4, 4, 0, 0, 0, 3)
    with pytest.raises(ValueError, match="group_size"):
        _lib.call("kvf_plan_init", p)
    p = _lib.kvf_plan(0, 8, 128, 1, 8, 1, 128, 4, 16, 4, 4, 0, 0, 0, 128)
    with pytest.raises(ValueError, match="T must be"):
        _lib.call("kvf_plan_init", p)


def test_restore_rejects_bad_frame_range_without_gpu():
    plan = L.plan_inter_frame(100, "R240", L.identity_layout(8, 128), 4)
    c = plan.to_c(128)
    surf = _lib.kvf_surface(1, 3 * plan.frame_h * plan.frame_w, plan.frame_h * plan.frame_w,
                            plan.frame_w)
    dst = _lib.kvf_paged()
    dst.block_size = 16
    dst.dtype = _lib.KVF_I8
    with pytest.raises(ValueError, match="frame range"):
        _lib.call("kvf_restore", surf, 0, plan.frame_count + 1, c, None, dst, None)
    dst.dtype = _lib.KVF_BF16
    with pytest.raises(ValueError, match="scales"):
        _lib.call("kvf_restore", surf, 0, 1, c, None, dst, None)
