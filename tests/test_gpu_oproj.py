"""The o_proj consumer: the tcgen05 GEMM with the fused
reduce-scatter epilogue, on one GPU.

* one rank: Y = O W stored, against torch's fp32 matmul of the same bf16 inputs;
* T virtual ranks on one device: rank r multiplies its head slice O[:, r] by its W_o
  rows and reduces every tile into the row owner's Y buffer (the buffers play the
  peer-mapped Ys of a real TP group); the assembled Y must equal the full O W.
Tolerance: fp32 accumulation of exact bf16 products, so only the summation order
differs: max |Y - Y_ref| <= 1e-4 * max |Y_ref|.
"""
import pytest
import torch

from paper_2410_18038_b200.tp import oproj

pytestmark = pytest.mark.gpu


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _inputs(tokens, k, n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    o = (torch.rand(tokens, k, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(k, n, generator=g, device="cuda") * 2 - 1) / 64).to(torch.bfloat16)
    return o, w, o.float() @ w.float()


@pytest.mark.parametrize("tokens,k,n", [(1088, 4096, 4096), (300, 512, 256), (1, 128, 128), (129, 1024, 384)])
def test_oproj_single_rank_matches_torch(tokens, k, n):
    _need_gpu()
    o, w, ref = _inputs(tokens, k, n, 1)
    y = torch.full((tokens, n), float("nan"), device="cuda")
    oproj(o, w, [y])
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    assert float((y - ref).abs().max()) <= 1e-4 * float(ref.abs().max())


@pytest.mark.parametrize("world", [2, 4, 8])
def test_oproj_reduce_scatter_virtual_ranks(world):
    _need_gpu()
    tokens, hq, d, n = 1088, 32, 128, 1024
    o, w, ref = _inputs(tokens, hq * d, n, 2)
    rows = (tokens + world - 1) // world
    ys = [torch.zeros(rows, n, device="cuda") for _ in range(world)]
    kr = hq * d // world
    for r in range(world):  # rank r: its q heads' columns of O and rows of W_o
        oproj(o[:, r * kr:(r + 1) * kr].contiguous(), w[r * kr:(r + 1) * kr].contiguous(), ys, rows_per_rank=rows,
              accumulate=True)
    torch.cuda.synchronize()
    y = torch.cat(ys)[:tokens]
    assert float((y - ref).abs().max()) <= 1e-4 * float(ref.abs().max())


def test_oproj_rejects_bad_shapes():
    _need_gpu()
    o = torch.zeros(4, 100, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(100, 128, dtype=torch.bfloat16, device="cuda")
    import paper_2410_18038_b200 as pkg

    with pytest.raises(pkg.Unsupported):
        oproj(o, w, [torch.zeros(4, 128, device="cuda")])
