"""Generates tests/golden/attention_golden.npz from the REFERENCE itself.

Runs the reference's own headers (compiled in place into oracle/_ref/ by
oracle/Makefile from /root/reference/proj/include) on the cases of
/root/reference/proj/tests/test_attention.cpp, with inputs drawn exactly as
those tests draw them (tests/golden/cases.py).  Only outputs (and the first
Rng draws, to pin the input generator) are stored, so the GPU box -- which has
no /root/reference -- can still pin the oracle port.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from oracle import pyoracle as O  # noqa: E402
import cases  # noqa: E402

OUT = Path(__file__).resolve().parent / "attention_golden.npz"


def main():
    g = {}
    for seed in (42, 43, 44, 2024, 4242):
        g[f"rng/{seed}"] = O.rng_doubles(seed, 64)
    q, k, v = cases.naive42()
    g["naive42/out"] = O.naive_attention(q, k, v, 2.0, which="ref")
    g["naive42/out_causal5"] = O.naive_attention(q, k, v, 2.0, causal_offset=5, which="ref")
    for gen in (cases.prefill_named, cases.prefill_random2024):
        for name, (chunk, ctx, off, hq, hkv, d), tiles, (q, k, v) in gen():
            for tq, tkv in tiles:
                g[f"{name}/out_{tq}_{tkv}"] = O.tiled_prefill(q, k, v, off, hq, hkv, np.sqrt(d), tq, tkv, which="ref")
            if name.startswith("p"):
                # prefill LSE via the reference's decode_attention_splitk on the prefix
                lse = np.zeros((chunk, hq))
                for r in range(chunk):
                    vis = off + r + 1
                    _, l, _ = O.decode_splitk(q[r], k[:vis], v[:vis], hq, hkv, np.sqrt(d), 1, which="ref")
                    lse[r] = l[0]
                g[f"{name}/lse"] = lse
    for gen in (cases.decode_named, cases.decode_random4242):
        for name, (ctx, hq, hkv, d), splits, (q, k, v) in gen():
            for s in splits:
                o, l, rg = O.decode_splitk(q, k, v, hq, hkv, np.sqrt(d), s, which="ref")
                g[f"{name}/lse_{s}"], g[f"{name}/rg_{s}"] = l, rg
                if not name.startswith("r"):
                    g[f"{name}/o_{s}"] = o
                g[f"{name}/merged_{s}"] = O.merge_partials(o, l, rg, which="ref")
    np.savez_compressed(OUT, **g)
    print(OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
