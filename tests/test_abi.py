"""The C-ABI library loads and exports every entry point include/pod_attn.h
declares; host-only calls behave (no GPU needed)."""
import ctypes as C
import re
from pathlib import Path

import pytest

import paper_2410_18038_b200 as pkg
from paper_2410_18038_b200 import _abi
from paper_2410_18038_b200.pod import GpuSpec, HybridBatchSpec, ModelShape, Plan, PlanOptions, PrefillSpec, DecodeSpec

HEADER = Path(__file__).resolve().parents[1] / "include" / "pod_attn.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:pod_status|void|size_t|char\s*\*|int)\s*\**\s*(pod_\w+)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pod_attn_plan", "pod_attn_run", "pod_attn_run_serial", "pod_attn_plan_destroy",
                 "pod_attn_workspace_bytes", "pod_attn_plan_tasks"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(_abi.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers the same set
    assert sorted(n for n, _, _ in _abi.SYMBOLS) == declared_functions()


def test_abi_version_and_status_strings():
    l = _abi.lib()
    assert l.pod_attn_abi_version() == 2
    for code, name in _abi.STATUS_NAMES.items():
        assert l.pod_status_string(code).decode() == name


def test_reference_default_device_matches_gpuspec():
    d = GpuSpec.reference_default()  # gpu.hpp:12-37
    assert (d.num_sms, d.compute_rate_per_sm, d.mem_bandwidth_total, d.mem_bandwidth_per_sm, d.mem_interference,
            d.max_ctas_per_sm, d.shared_mem_per_sm) == (108, 0.25, 108.0, 1.2, 0.25, 4, 167936.0)


def test_plan_info_and_workspace():
    shape = ModelShape(32, 8, 128, 128 ** 0.5)
    b = HybridBatchSpec(prefill=PrefillSpec(1024, 16384, 15360), decodes=[DecodeSpec(16384)] * 64, shape=shape)
    # default: warp-specialised one-CTA-per-SM kernel (two-block prefill items; decode
    # parents split in 2; the last request's 8 parents in 3, filling the 7th wave of 148
    # items as far as whole requests allow: 1032 of 1036)
    p = Plan(b, GpuSpec.b200())
    i = p.info()
    assert i.num_prefill_ctas == 128 and i.num_decode_ctas == 1032 and i.decode_splits == 3
    assert 6 * 148 < i.num_decode_ctas <= 7 * 148
    assert i.smem_bytes > 0 and p.workspace_bytes() == i.workspace_bytes > 0
    assert i.smem_bytes + 1024 <= 233472  # one CTA per SM
    # the pair engine's tile width: 32 keys for this decode-dominant batch, forceable
    assert i.prefill_tile_keys == 32
    assert Plan(b, GpuSpec.b200(), PlanOptions(prefill_tile_keys=64)).info().prefill_tile_keys == 64
    assert i.prefill_s_buffers == 2  # the 32-key engine double-buffers S
    for sb in (1, 2):  # the 64-key engine: one S buffer (Q in TMEM) or two (Q in smem, own kernel instance)
        isb = Plan(b, GpuSpec.b200(), PlanOptions(prefill_tile_keys=64, prefill_s_buffers=sb)).info()
        assert isb.prefill_s_buffers == sb and isb.smem_bytes + 1024 <= 233472
    # the two-CTA-per-SM POD kernel
    p = Plan(b, GpuSpec.b200(), PlanOptions(policy=_abi.POD_POLICY_COMPLEMENT))
    i = p.info()
    assert i.num_prefill_ctas == 256 and i.num_decode_ctas == 512
    assert 2 * (i.smem_bytes + 1024) <= 233472  # two CTAs per SM


def test_error_codes_cross_the_boundary_as_statuses():
    with pytest.raises(pkg.InvalidArgument):
        Plan(HybridBatchSpec(shape=ModelShape(32, 8, 128, 1.0)), GpuSpec.b200())
    with pytest.raises(pkg.InvalidArgument):
        Plan(HybridBatchSpec(decodes=[DecodeSpec(5)], shape=ModelShape(32, 8, 128, 1.0)), GpuSpec(num_sms=0))
    with pytest.raises(pkg.InvalidArgument):  # pair-engine tile width other than 0 / 32 / 64
        Plan(HybridBatchSpec(decodes=[DecodeSpec(5)], shape=ModelShape(32, 8, 128, 1.0)), GpuSpec.b200(),
             PlanOptions(prefill_tile_keys=48))
    with pytest.raises(pkg.InvalidArgument):  # out_dtype outside POD_OUT_*
        Plan(HybridBatchSpec(decodes=[DecodeSpec(5)], shape=ModelShape(32, 8, 128, 1.0)), GpuSpec.b200(),
             PlanOptions(out_dtype=3))
    # run entry points validate arguments before touching CUDA
    st = _abi.lib().pod_attn_run(None, None, None, None, None, 0, None, None, None, None, None, None, None, None)
    assert st == 1


def test_unsupported_shapes_are_reported_not_faked():
    # any head_dim plans (host semantics); the sm_100a kernels run d = 8..128 in steps of 8
    # (zero-padded to 128: 16-byte TMA row strides), so d = 4, 12 or 256 is reported, before CUDA
    for d in (4, 12, 256):
        b = HybridBatchSpec(decodes=[DecodeSpec(100)], shape=ModelShape(8, 2, d, 8.0))
        p = Plan(b, GpuSpec.b200())
        st = _abi.lib().pod_attn_run(p.handle, None, C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), 1,
                                     C.c_void_p(16), C.c_void_p(16), None, None, C.c_void_p(16), C.c_void_p(16),
                                     C.c_void_p(16), None)
        assert st == 7, d  # POD_ERR_UNSUPPORTED
