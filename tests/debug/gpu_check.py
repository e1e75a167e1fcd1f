"""Debug driver: runs hybrid-batch cases in subprocesses and prints oracle errors."""
import json, subprocess, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

CASES = {
    "decode_small": dict(hq=32, hkv=8, chunk=0, offset=0, dec=[300, 77, 1024, 16, 1], modes=["decode", "fused"]),
    "prefill_small": dict(hq=32, hkv=8, chunk=96, offset=160, dec=[], modes=["prefill", "fused"]),
    "hybrid_small": dict(hq=32, hkv=8, chunk=96, offset=160, dec=[300, 77, 1024], modes=["serial", "fused"]),
    "hybrid_ref_tiles": dict(hq=32, hkv=8, chunk=200, offset=37, dec=[500, 33], modes=["fused"], tile_mode=0),
    "mha": dict(hq=8, hkv=8, chunk=130, offset=0, dec=[257, 64], modes=["fused"]),
    "c1": dict(hq=32, hkv=8, chunk=512, offset=1536, dec=[2048] * 8, modes=["fused", "serial"], heads=[0, 5], reqs=[0, 7]),
}

def run_case(name):
    import numpy as np, torch
    import paper_2410_18038_b200 as pkg
    from paper_2410_18038_b200.hybrid import PodAttention
    from paper_2410_18038_b200.workload import build_workload, make_batch
    from tests.common import compare_decode, compare_prefill
    c = CASES[name]
    shape = pkg.ModelShape(c["hq"], c["hkv"], 128, 128 ** 0.5)
    batch = make_batch(shape, chunk=c["chunk"], offset=c["offset"], decode_ctx=c["dec"])
    wl = build_workload(batch, device="cuda")
    import os
    opts = pkg.PlanOptions(tile_mode=c.get("tile_mode", 1), policy=int(os.environ.get("POD_POLICY", "3")))
    op = PodAttention(batch, options=opts)
    info = op.info
    res = {"P": info.num_prefill_ctas, "D": info.num_decode_ctas, "splits": info.prefill_splits,
           "dsplits": info.decode_splits}
    for mode in c["modes"]:
        t0 = time.time()
        out = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, mode=mode)
        torch.cuda.synchronize()
        r = {}
        if batch.prefill is not None and mode in ("prefill", "fused", "serial"):
            r["pf"] = compare_prefill(wl, out.o_prefill.cpu().numpy(), out.lse_prefill.cpu().numpy(), kv_heads=c.get("heads"))
        if batch.decodes and mode in ("decode", "fused", "serial"):
            r["dec"] = compare_decode(wl, out.o_decode.cpu().numpy(), out.lse_decode.cpu().numpy(), requests=c.get("reqs"))
        r["t"] = round(time.time() - t0, 2)
        res[mode] = r
    print("RESULT", name, json.dumps(res))

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] in CASES:
        run_case(sys.argv[1]); sys.exit(0)
    for name in CASES:
        p = subprocess.run([sys.executable, __file__, name], capture_output=True, text=True, timeout=600)
        lines = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        print(lines[0] if lines else f"FAIL {name} rc={p.returncode}\n{p.stderr[-3000:]}", flush=True)
