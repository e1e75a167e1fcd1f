"""Per-tile timeline of the 64-key pair engine (CTA 0, first prefill item), from a
POD_TRACE_STAMPS build:

  tools/micro/build_variant.sh trace -DPOD_TRACE_STAMPS=1
  POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1 python tools/trace64.py [--config c2_b8] [--mode prefill]

Stamps (clock64 low words, SM-local cycles): row t = block A, row 384 + t = block B
  k0 softmax waits S(t) | k1 S(t) ready | k2 warp 0 arrived P(t) | k3 warp 3 arrived
  k4 MMA saw P_X(t)     | k5 MMA issued PV_X(t) + QK_X(t+1)
  row B k6 / k7: producer issued K(t) / V(t)
Prints the steady-state median of each interval (tiles 16 .. nt-16)."""
import argparse
import math
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2410_18038_b200 as pkg  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2_b8")
    ap.add_argument("--mode", default="prefill")
    ap.add_argument("--precision", type=int, default=2)
    ap.add_argument("--keys", type=int, default=64)
    ap.add_argument("--raw", action="store_true", help="print the first tiles' raw stamps")
    ap.add_argument("--chunk", type=int, default=0, help="override the config's chunk (32 rows x G=4 = one M-block)")
    a = ap.parse_args()
    assert os.environ.get("POD_TRACE"), "set POD_TRACE=1 with a POD_TRACE_STAMPS build (POD_LIB)"
    hq, hkv, chunk, off, b, ctx = CONFIGS[a.config]
    if a.chunk:
        off, chunk = off + chunk - a.chunk, a.chunk
    batch = make_batch(pkg.ModelShape(hq, hkv, 128, math.sqrt(128)), chunk=chunk, offset=off, decode_ctx=[ctx] * b)
    wl = build_workload(batch, device="cuda")
    gpu = pkg.GpuSpec.from_device(0)
    if a.chunk:  # one item per KV head, unsplit: plan for as many SMs as items
        import dataclasses
        gpu = dataclasses.replace(gpu, num_sms=hkv)
    op = PodAttention(batch, gpu=gpu,
                      options=pkg.PlanOptions(policy=7, prefill_tile_keys=a.keys, precision=a.precision))
    log = op.enable_role_log(768 * 8)
    out = op.alloc_outputs()
    for _ in range(2):
        log.zero_()
        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=out, mode=a.mode)
    torch.cuda.synchronize()
    nrec = int(op.info.num_prefill_ctas + op.info.num_decode_ctas)
    tr = log.view(-1, 8)[nrec:].cpu().long() & 0xffffffff
    A, B = tr[:384], tr[384:768]
    nt = int((A[:, 1] != 0).sum())
    print(f"{a.config} chunk {chunk} {a.mode} precision {a.precision} keys {a.keys}: "
          f"{nt} tiles traced")
    if nt < 40 or a.raw:
        # raw timeline of the first tiles, cycles from block A's first S wait:
        # A: k0 wait S, k1 S ready, k2 w0 arrive P, k4 MMA saw P_A, k5 MMA issued; B: same; producer K / V issue
        base = int(A[0, 0])
        rel = lambda x: ((int(x) - base) & 0xffffffff) if int(x) else None  # noqa: E731
        for t in sorted(set(range(min(nt, 4))) | set(range(max(nt - 3, 0), nt))):
            print(f"  t{t}: A {[rel(A[t, k]) for k in (0, 1, 2, 4, 5)]} B {[rel(B[t, k]) for k in (0, 1, 2, 4, 5)]} "
                  f"prod K/V {[rel(B[t, 6]), rel(B[t, 7])]}")
        F = tr[766]
        print(f"  epilogue w0: before PV wait {rel(F[0])}, PV done {rel(F[1])}, chunk lds {[rel(F[k]) for k in range(2, 6)]}")
        E = tr[767]
        print(f"  CTA entry {rel(E[0])}, item claimed {rel(E[1])}, softmax w0 done {rel(E[2])}, "
              f"producer done {rel(E[3])}, MMA done {rel(E[4])}")
        if nt < 40:
            return
    rng = range(16, nt - 16)

    def med(xs):
        xs = sorted(xs)
        return xs[len(xs) // 2]

    def d(x, y):  # y - x with 32-bit wrap
        return (y - x) & 0xffffffff

    if a.keys == 32:  # the 32-key double-S engine's stamps (pod_sm.cuh)
        rng = range(16, min(nt, 128) - 16)
        rows32 = {
            "period per 32-key tile (S_A(t) ready -> S_A(t+1) ready)": [d(A[t, 1], A[t + 1, 1]) for t in rng],
            "A softmax (S ready -> warp0 arrive)": [d(A[t, 1], A[t, 2]) for t in rng],
            "A waits S (k0 -> k1)": [d(A[t, 0], A[t, 1]) for t in rng],
            "A arrive(w3) -> MMA sees P_A": [d(A[t, 3], A[t, 4]) for t in rng],
            "MMA: P_A seen -> PV_A committed": [d(A[t, 4], A[t, 5]) for t in rng],
            "MMA: PV_A committed -> QK_A(t+2) committed": [d(A[t, 5], A[t, 6]) for t in rng],
            "B softmax": [d(B[t, 1], B[t, 2]) for t in rng],
            "B waits S": [d(B[t, 0], B[t, 1]) for t in rng],
        }
        for k, v in rows32.items():
            print(f"  {k:55s} {med(v):6d} cyc")
        return
    rows = {
        "period (S_A(t) ready -> S_A(t+1) ready)": [d(A[t, 1], A[t + 1, 1]) for t in rng],
        "A softmax (S ready -> warp0 arrive)": [d(A[t, 1], A[t, 2]) for t in rng],
        "A warp spread (w0 -> w3 arrive)": [d(A[t, 2], A[t, 3]) for t in rng],
        "A arrive(w3) -> MMA sees P_A": [d(A[t, 3], A[t, 4]) for t in rng],
        "MMA issue PV_A + QK_A": [d(A[t, 4], A[t, 5]) for t in rng],
        "QK_A(t+1) issued -> S_A(t+1) ready": [d(A[t, 5], A[t + 1, 1]) for t in rng],
        "A waits S (k0 -> k1)": [d(A[t, 0], A[t, 1]) for t in rng],
        "  A: S ready -> S in registers (tcgen05.ld)": [d(A[t, 1], A[t, 6]) for t in rng],
        "  A: max, rescale check, exp, P pack + tcgen05.st": [d(A[t, 6], A[t, 7]) for t in rng],
        "  A: wait::st, fence, syncwarp -> arrive": [d(A[t, 7], A[t, 2]) for t in rng],
        "B softmax": [d(B[t, 1], B[t, 2]) for t in rng],
        "B arrive(w3) -> MMA sees P_B": [d(B[t, 3], B[t, 4]) for t in rng],
        "MMA issue PV_B + QK_B": [d(B[t, 4], B[t, 5]) for t in rng],
        "QK_B(t+1) issued -> S_B(t+1) ready": [d(B[t, 5], B[t + 1, 1]) for t in rng],
        "B waits S": [d(B[t, 0], B[t, 1]) for t in rng],
        "MMA: PV_A issued -> sees P_B": [d(A[t, 5], B[t, 4]) for t in rng],
        "MMA: QK_B issued -> sees P_A(t+1)": [d(B[t, 5], A[t + 1, 4]) for t in rng],
        "producer K(t) issued ahead of S_A(t) ready": [d(B[t, 6], A[t, 1]) for t in rng],
    }
    for k, v in rows.items():
        if "B" in k.split(" ")[0] or "P_B" in k or "QK_B" in k or "PV_B" in k:
            if not int((B[:, 1] != 0).sum()):
                continue
        print(f"  {k:45s} {med(v):6d} cyc")


if __name__ == "__main__":
    main()
