"""GPU kernel unit tests: each CUDA kernel against a plain PyTorch fp32 reference of the same op on the
same (dtype-rounded) inputs."""
import numpy as np
import pytest
import torch

from paper_2410_07590_b200 import turbokv as T

pytestmark = pytest.mark.gpu


def bf16_round(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy()


GEMM_SHAPES = [(32, 96, 64), (64, 128, 64), (128, 128, 128), (200, 300, 192), (1, 259, 64), (64, 4608, 3584),
               (129, 520, 1000), (8256, 512, 3584)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
@pytest.mark.parametrize("use_tc,dtype", [(True, "bf16"), (False, "bf16"), (False, "f32")])
def test_gemm_vs_torch(M, N, K, use_tc, dtype):
    if M * N * K > 8256 * 512 * 3584 // 2 and not use_tc:
        pytest.skip("large SIMT case covered by the tcgen05 run")
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    if dtype == "bf16":
        A, W = bf16_round(A), bf16_round(W)
    ref = (torch.from_numpy(A).double() @ torch.from_numpy(W).double().T).numpy()
    for splits in (1, 3):
        out = T.debug_gemm(A, W, dtype=dtype, use_tc=use_tc, splits=splits)
        err = np.abs(out - ref).max() / np.abs(ref).max()
        assert err < 1e-5, f"splits={splits}: max rel err {err:.3e}"


def attention_ref(q, k, v, lo, hi, H, Hkv, d):
    Tq, Tk = q.shape[0], k.shape[0]
    g = H // Hkv
    qh = torch.from_numpy(q).double().view(Tq, H, d)
    kh = torch.from_numpy(k).double().view(Tk, Hkv, d).repeat_interleave(g, dim=1)
    vh = torch.from_numpy(v).double().view(Tk, Hkv, d).repeat_interleave(g, dim=1)
    s = torch.einsum("qhd,khd->hqk", qh, kh) / np.sqrt(d)
    j = torch.arange(Tk)[None, :]
    vis = (j >= torch.from_numpy(np.asarray(lo))[:, None]) & (j <= torch.from_numpy(np.asarray(hi))[:, None])
    s = s.masked_fill(~vis[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, vh).reshape(Tq, H * d).numpy()


ATTN_CASES = [
    # (Tq, Tk, H, Hkv, d, kind)
    (32, 544, 8, 2, 8, "query"),      # C1 query prefill
    (544, 544, 8, 2, 8, "indep"),     # C1 naive independent
    (64, 8256, 28, 4, 128, "query"),  # C2 query prefill
    (300, 300, 28, 4, 128, "causal"),
    (700, 700, 28, 4, 128, "indep"),
    (5, 1030, 32, 8, 128, "query"),
    (1, 8256, 28, 4, 128, "query"),     # last-layer tail row (splits = 32)
    (37, 2000, 32, 8, 128, "query"),    # group 4: 148 rows -> tile B partially filled
    (64, 3000, 28, 4, 128, "query_hot"),  # large scores: exercises the lazy O rescale
    (20, 20, 28, 4, 128, "causal"),     # one key tile, heavy masking
    # compact last row tile (<= 64 valid rows: 16 per TMEM quadrant, half the softmax warps) with the split plan
    (48, 4000, 32, 8, 128, "query"),    # group 4: 192 rows -> last tile exactly 64 rows (compact)
    (192, 2500, 4, 4, 128, "query"),    # group 1: 192 rows -> last tile 64 rows (compact)
    (193, 2500, 4, 4, 128, "query"),    # group 1: 193 rows -> last tile 65 rows (not compact)
]


@pytest.mark.parametrize("Tq,Tk,H,Hkv,d,kind", ATTN_CASES)
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_attention_vs_torch(Tq, Tk, H, Hkv, d, kind, dtype):
    rng = np.random.default_rng(Tq + Tk + d)
    q = rng.uniform(-1, 1, (Tq, H * d)).astype(np.float32)
    k = rng.uniform(-1, 1, (Tk, Hkv * d)).astype(np.float32)
    v = rng.uniform(-1, 1, (Tk, Hkv * d)).astype(np.float32)
    if dtype == "bf16":
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    if kind == "query_hot":
        # growing score scale along the keys forces the running max up tile after tile
        q = q * 6.0
        k = k * np.linspace(0.2, 1.5, Tk, dtype=np.float32)[:, None]
        if dtype == "bf16":
            q, k = bf16_round(q), bf16_round(k)
    if kind.startswith("query"):
        P = Tk - Tq
        lo, hi = np.zeros(Tq, np.int32), (P + np.arange(Tq)).astype(np.int32)
    elif kind == "causal":
        lo, hi = np.zeros(Tq, np.int32), np.arange(Tq, dtype=np.int32)
    else:  # chunks of 128 + final query segment of 32
        starts = np.minimum(np.arange(Tq) // 128 * 128, Tq - 32)
        lo = np.where(np.arange(Tq) >= Tq - 32, 0, starts).astype(np.int32)
        hi = np.arange(Tq, dtype=np.int32)
    out = T.debug_attention(q, k, v, lo, hi, H, Hkv, d, dtype=dtype)
    ref = attention_ref(q, k, v, lo, hi, H, Hkv, d)
    tol = 1e-5 if dtype == "f32" else 1e-2
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < tol, f"max rel err {err:.3e}"


def test_attention_degenerate_row_raises():
    q = np.ones((2, 8), np.float32)
    k = np.ones((4, 8), np.float32)
    with pytest.raises(T.DegenerateRowError):
        T.debug_attention(q, k, k, [0, 3], [1, 2], 1, 1, 8, dtype="f32")


DECODE_CASES = [
    # (Tq, Tk, H, Hkv, kind): the last layer's single row, greedy-decode steps, small query tails
    (1, 8256, 28, 4, "query"),
    (2, 1000, 32, 8, "query"),   # 8 rows per kv head
    (1, 7, 28, 4, "query"),
    (2, 3000, 28, 4, "query_hot"),  # 14 rows -> not a decode shape: tcgen05 path (skipped below)
    (1, 5000, 64, 4, "query_hot"),  # 16 rows per kv head, growing scores
    (1, 300, 32, 8, "query"),    # 4 rows per kv head
]


@pytest.mark.parametrize("Tq,Tk,H,Hkv,kind", DECODE_CASES)
def test_decode_attention_vs_torch(Tq, Tk, H, Hkv, kind):
    d = 128
    if Tq * (H // Hkv) not in (4, 7, 8, 16):
        pytest.skip("not a decode-sized row count")
    rng = np.random.default_rng(Tq * 7 + Tk + H)
    q = rng.uniform(-1, 1, (Tq, H * d)).astype(np.float32)
    k = rng.uniform(-1, 1, (Tk, Hkv * d)).astype(np.float32)
    v = bf16_round(rng.uniform(-1, 1, (Tk, Hkv * d)).astype(np.float32))
    if kind == "query_hot":
        q = q * 6.0
        k = k * np.linspace(0.2, 1.5, Tk, dtype=np.float32)[:, None]
    q, k = bf16_round(q), bf16_round(k)
    P = Tk - Tq
    lo, hi = np.zeros(Tq, np.int32), (P + np.arange(Tq)).astype(np.int32)
    out = T.debug_attention(q, k, v, lo, hi, H, Hkv, d, dtype="bf16", impl=2)
    ref = attention_ref(q, k, v, lo, hi, H, Hkv, d)
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < 1e-2, f"max rel err {err:.3e}"
