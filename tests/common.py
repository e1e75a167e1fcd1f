"""Shared checking helpers: run the CPU oracle (oracle/pyoracle.py, test
infrastructure) on the same bf16 inputs the GPU receives and compare."""
from __future__ import annotations

import sys
from pathlib import Path
from typing import Dict, Iterable, Optional

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import pyoracle as O  # noqa: E402

# North-star tolerance: fp32 accumulate, bf16 inputs -> max abs error <= 2e-3
# relative to the output scale (max |O_ref| of the compared block); LSE is a
# natural log, compared absolutely.
O_TOL = 2e-3
LSE_TOL = 2e-3


def oracle_prefill(wl, kv_heads: Optional[Iterable[int]] = None, row_range=None) -> Dict[int, tuple]:
    """Per kv head h: (O [rows][G][d], lse [rows][G]) from the oracle port of
    tiled_prefill_attention (attention.hpp:148-222) on a one-KV-head restriction
    (GQA consistency, test_attention.cpp:252-270)."""
    s = wl.batch.shape
    G = s.group_size()
    off = wl.batch.prefill.position_offset
    q = wl.prefill_q().numpy()
    r0, r1 = row_range if row_range else (0, q.shape[0])
    out = {}
    for h in (kv_heads if kv_heads is not None else range(s.num_kv_heads)):
        ctx = off + r1
        k = wl.request_cache(0, "k", head=h)[:ctx].numpy().reshape(ctx, 1, s.head_dim)
        v = wl.request_cache(0, "v", head=h)[:ctx].numpy().reshape(ctx, 1, s.head_dim)
        qh = np.ascontiguousarray(q[r0:r1, h * G:(h + 1) * G, :])
        o = O.tiled_prefill(qh, k, v, off + r0, G, 1, s.scale, 64, 64)
        lse = O.prefill_lse(qh, k, off + r0, G, 1, s.scale)
        out[h] = (o, lse)
    return out


def oracle_decode(wl, requests: Optional[Iterable[int]] = None, kv_heads=None) -> Dict[tuple, tuple]:
    """(request, kv head) -> (O [G][d], lse [G]) from decode_attention (attention.hpp:328-333)."""
    s = wl.batch.shape
    G = s.group_size()
    q = wl.decode_q().numpy()
    base = 1 if wl.batch.prefill is not None else 0
    out = {}
    reqs = requests if requests is not None else range(len(wl.batch.decodes))
    for r in reqs:
        for h in (kv_heads if kv_heads is not None else range(s.num_kv_heads)):
            ctx = wl.kv_lens[base + r]
            k = wl.request_cache(base + r, "k", head=h).numpy().reshape(ctx, 1, s.head_dim)
            v = wl.request_cache(base + r, "v", head=h).numpy().reshape(ctx, 1, s.head_dim)
            o, lse = O.decode_attention(np.ascontiguousarray(q[r, h * G:(h + 1) * G]), k, v, G, 1, s.scale)
            out[(r, h)] = (o, lse)
    return out


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    scale = max(float(np.abs(ref).max()), 1e-30)
    return float(np.abs(got - ref).max()) / scale


def compare_prefill(wl, o_gpu: np.ndarray, lse_gpu: np.ndarray, kv_heads=None, row_range=None):
    """Returns (worst O rel err, worst |dLSE|)."""
    G = wl.batch.shape.group_size()
    ref = oracle_prefill(wl, kv_heads, row_range)
    r0, r1 = row_range if row_range else (0, o_gpu.shape[0])
    eo = el = 0.0
    for h, (o, lse) in ref.items():
        got = o_gpu[r0:r1, h * G:(h + 1) * G, :]
        eo = max(eo, rel_err(got, o))
        el = max(el, float(np.abs(lse_gpu[r0:r1, h * G:(h + 1) * G] - lse).max()))
    return eo, el


def compare_decode(wl, o_gpu: np.ndarray, lse_gpu: np.ndarray, requests=None, kv_heads=None):
    G = wl.batch.shape.group_size()
    ref = oracle_decode(wl, requests, kv_heads)
    eo = el = 0.0
    for (r, h), (o, lse) in ref.items():
        eo = max(eo, rel_err(o_gpu[r, h * G:(h + 1) * G], o))
        el = max(el, float(np.abs(lse_gpu[r, h * G:(h + 1) * G] - lse).max()))
    return eo, el


def new_token_rows(wl):
    """The batch's new K/V rows as the KV-append step receives them (16-bit words):
    prefill tokens = positions [offset, offset + chunk) of request 0, decode b's token
    = position ctx_b - 1 of its request.  Returns (kp, vp, kd, vd) as uint16 arrays
    [chunk][Hkv][d] / [B][Hkv][d] (None when absent), read from the HND pool at the
    tokens' (page, slot) -- exactly the cached bits, for any 16-bit dtype."""
    import torch

    kb = wl.k_pool.cpu().view(torch.int16).numpy().view(np.uint16)
    vb = wl.v_pool.cpu().view(torch.int16).numpy().view(np.uint16)
    slots = token_slots(wl)
    k = np.stack([kb[page, :, slot, :] for page, slot in slots])
    v = np.stack([vb[page, :, slot, :] for page, slot in slots])
    c = wl.batch.prefill.chunk_size if wl.batch.prefill is not None else 0
    kp, vp = (k[:c], v[:c]) if c else (None, None)
    kd, vd = (k[c:], v[c:]) if wl.batch.decodes else (None, None)
    return kp, vp, kd, vd


def token_slots(wl):
    """(page, slot) of every new token, prefill first then decodes (HND pool indexing)."""
    ip, ix = wl.page_indptr.cpu().tolist(), wl.page_indices.cpu().tolist()
    b = wl.batch
    out, base = [], 0
    if b.prefill is not None:
        off, c = b.prefill.position_offset, b.prefill.chunk_size
        out += [(ix[ip[0] + t // 16], t % 16) for t in range(off, off + c)]
        base = 1
    for i, d in enumerate(b.decodes):
        t = d.context_len - 1
        out.append((ix[ip[base + i] + t // 16], t % 16))
    return out


def dense_layer(wl):
    """The whole layer as float64 dense attention (torch, on the workload's device): O
    [chunk + B][Hq][d] and natural-log LSE [chunk + B][Hq], prefill rows first.  K / V
    are gathered from the paged pools through the block table (HND), so this checks the
    sharded pools and tables too.  Semantics: attention.hpp:148-222 (row r of the chunk
    sees keys [0, offset + r]) and :240-333 (a decode sees all ctx keys)."""
    import torch

    b, s = wl.batch, wl.batch.shape
    G, d = s.group_size(), s.head_dim
    ip = wl.page_indptr.tolist()

    def kv(req):
        ctx = wl.kv_lens[req]
        pages = wl.page_indices[ip[req]:ip[req + 1]].long()
        k = wl.k_pool[pages].permute(0, 2, 1, 3).reshape(-1, s.num_kv_heads, d)[:ctx].double()
        v = wl.v_pool[pages].permute(0, 2, 1, 3).reshape(-1, s.num_kv_heads, d)[:ctx].double()
        return k, v

    def attend(q, k, v, limit):  # q [m][Hq][d], k/v [n][Hkv][d], row i sees keys <= limit[i]
        kk = k.repeat_interleave(G, dim=1)
        vv = v.repeat_interleave(G, dim=1)
        sc = torch.einsum("mhd,nhd->hmn", q, kk) / s.scale
        j = torch.arange(k.shape[0], device=q.device)
        sc = sc.masked_fill(j[None, None, :] > limit[None, :, None], float("-inf"))
        lse = torch.logsumexp(sc, dim=-1)
        o = torch.einsum("hmn,nhd->mhd", torch.softmax(sc, dim=-1), vv)
        return o, lse.transpose(0, 1)

    os_, ls_ = [], []
    base = 0
    if b.prefill is not None:
        k, v = kv(0)
        c, off = b.prefill.chunk_size, b.prefill.position_offset
        o, lse = attend(wl.q_prefill.double(), k, v, off + torch.arange(c, device=k.device))
        os_.append(o)
        ls_.append(lse)
        base = 1
    for i in range(len(b.decodes)):
        k, v = kv(base + i)
        o, lse = attend(wl.q_decode[i:i + 1].double(), k, v, torch.tensor([k.shape[0] - 1], device=k.device))
        os_.append(o)
        ls_.append(lse)
    return torch.cat(os_), torch.cat(ls_)
