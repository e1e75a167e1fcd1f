"""Input recipes of the reference's attention tests
(/root/reference/proj/tests/test_attention.cpp), reproduced with the Python
splitmix64 Rng so fixtures only need to store outputs.  Shared by
make_golden.py (writer, runs the reference) and tests/test_oracle.py (reader)."""
import numpy as np

from paper_2410_18038_b200.workload import Rng


def prefill_case(rng, chunk, ctx, off, hq, hkv, d):
    # random_prefill_case (test_attention.cpp:64-74): q, then k, then v.
    q = rng.fill_uniform(chunk * hq * d).numpy().reshape(chunk, hq, d)
    k = rng.fill_uniform(ctx * hkv * d).numpy().reshape(ctx, hkv, d)
    v = rng.fill_uniform(ctx * hkv * d).numpy().reshape(ctx, hkv, d)
    return q, k, v


def decode_case(rng, ctx, hq, hkv, d):
    # random_decode_case (test_attention.cpp:280-289)
    q = rng.fill_uniform(hq * d).numpy().reshape(hq, d)
    k = rng.fill_uniform(ctx * hkv * d).numpy().reshape(ctx, hkv, d)
    v = rng.fill_uniform(ctx * hkv * d).numpy().reshape(ctx, hkv, d)
    return q, k, v


def naive42():
    # test_attention.cpp:131-142 (random_mat fills row-major)
    rng = Rng(42)
    q = rng.fill_uniform(32).numpy().reshape(8, 4)
    k = rng.fill_uniform(64).numpy().reshape(16, 4)
    v = rng.fill_uniform(64).numpy().reshape(16, 4)
    return q, k, v


# (name, seed, chunk, ctx, off, hq, hkv, d, [(tile_q, tile_kv)])
PREFILL_NAMED = [
    ("p11", 11, 1, 1, 0, 2, 1, 8, [(4, 1), (4, 7), (4, 64)]),   # :192-196
    ("p123", 123, 64, 512, 448, 4, 2, 16, [(16, 32)]),          # :198-202
    ("p5", 5, 12, 48, 36, 2, 2, 8, [(12, 1024)]),               # :204-208
    ("p99", 99, 6, 40, 20, 2, 1, 8, [(3, 8)]),                  # :229-244
    ("p31", 31, 10, 32, 16, 8, 2, 8, [(4, 8)]),                 # :252-270
]


def prefill_named():
    for name, seed, chunk, ctx, off, hq, hkv, d, tiles in PREFILL_NAMED:
        q, k, v = prefill_case(Rng(seed), chunk, ctx, off, hq, hkv, d)
        yield name, (chunk, ctx, off, hq, hkv, d), tiles, (q, k, v)


def prefill_random2024():
    # test_attention.cpp:210-227
    rng = Rng(2024)
    tiles = [1, 8, 16, 64, 128]
    for it in range(25):
        d = [4, 8, 64][rng.next_long(0, 2)]
        hkv = rng.next_long(1, 2)
        hq = hkv * rng.next_long(1, 2)
        chunk = rng.next_long(1, 64)
        off = rng.next_long(0, 512)
        ctx = off + chunk + rng.next_long(0, 64)
        q, k, v = prefill_case(rng, chunk, ctx, off, hq, hkv, d)
        tq = tiles[rng.next_long(0, 4)]
        tkv = tiles[rng.next_long(0, 4)]
        yield f"r2024_{it}", (chunk, ctx, off, hq, hkv, d), [(tq, tkv)], (q, k, v)


# (name, seed, ctx, hq, hkv, d, splits)
DECODE_NAMED = [("d8", 8, 24, 4, 2, 8, [1]), ("d3", 3, 12, 2, 1, 4, [4]), ("d77", 77, 1024, 4, 2, 16, [1, 2, 4, 8]),
                ("d6", 6, 5, 2, 1, 4, [64]), ("d9", 9, 10, 2, 1, 4, [1]), ("d21", 21, 37, 4, 2, 8, [4])]


def decode_named():
    for name, seed, ctx, hq, hkv, d, splits in DECODE_NAMED:
        q, k, v = decode_case(Rng(seed), ctx, hq, hkv, d)
        yield name, (ctx, hq, hkv, d), splits, (q, k, v)


def decode_random4242():
    # test_attention.cpp:336-348
    rng = Rng(4242)
    for it in range(20):
        d = [4, 8, 64][rng.next_long(0, 2)]
        kv = rng.next_long(1, 2)
        ctx = rng.next_long(8, 300)
        q, k, v = decode_case(rng, ctx, kv * 2, kv, d)
        yield f"r4242_{it}", (ctx, kv * 2, kv, d), list(range(1, 9)), (q, k, v)
