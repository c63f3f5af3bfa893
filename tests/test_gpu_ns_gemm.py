"""-m gpu: the tcgen05 Newton-Schulz GEMM (rsdb_ns_gemm_bf16, N3 / Alg. 2
l.10, reading R22) against a plain PyTorch fp32 reference of the same op.

C = alpha A B^T + beta D with bf16 A, B, D: every product of two bf16 values
is exact in fp32, so the fp32 reference differs from the kernel's fp32
accumulation only by summation order (<= K 2^-24 sum|a b| each way), and the
kernel rounds once to bf16 (half an ulp, 2^-8 relative).  Bound per element:
|C - ref| <= 2^-8 |ref| + 2 K 2^-24 (|alpha| sum_k |a b| + |beta d|) + tiny.
CT must equal C^T bit for bit.  Shapes cover one tile, several tiles and
k-blocks, ragged M / N / K edges (TMA zero fill), padded leading dimensions,
and the three GEMMs of one quintic iteration on a Llama-3-8B-sized matrix.
"""
import pytest
import torch

import paper_2602_22437_b200 as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _ld(cols, pad):
    return (cols + 7) // 8 * 8 + pad


def _mat(rows, cols, ld, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    buf = torch.randn(rows, ld, device="cuda", generator=g) * scale
    return buf.to(torch.bfloat16)[:, :cols]


def _check(M, N, K, alpha=1.0, beta=0.0, with_t=False, pad=0, seed=0):
    A = _mat(M, K, _ld(K, pad), seed)
    B = _mat(N, K, _ld(K, pad), seed + 1)
    D = _mat(M, N, _ld(N, pad), seed + 2) if beta != 0.0 else None
    C = torch.full((M, _ld(N, pad)), float("nan"), device="cuda", dtype=torch.bfloat16)[:, :N]
    CT = torch.zeros(N, _ld(M, pad), device="cuda", dtype=torch.bfloat16)[:, :M] if with_t else None
    R.ns_gemm_bf16(A, B, C, alpha, beta, D, CT)
    torch.cuda.synchronize()
    ref = alpha * (A.float() @ B.float().T)
    mag = abs(alpha) * (A.float().abs() @ B.float().abs().T)
    if D is not None:
        ref = ref + beta * D.float()
        mag = mag + abs(beta) * D.float().abs()
    err = (C.float() - ref).abs()
    bound = 2.0 ** -8 * ref.abs() + 2 * K * 2.0 ** -24 * mag + 1e-30
    assert torch.isfinite(C.float()).all()
    worst = (err / bound).max().item()
    assert worst <= 1.0, (M, N, K, worst)
    if with_t:
        assert torch.equal(CT.contiguous().view(torch.int16), C.T.contiguous().view(torch.int16))


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (384, 768, 4096 + 64)])
def test_ns_gemm_full_tiles(M, N, K):
    _check(M, N, K)


@pytest.mark.parametrize("M,N,K,pad", [(24, 40, 24, 0), (200, 300, 136, 8), (1, 64, 8, 0), (130, 260, 72, 16),
                                       (1000, 1000, 1000, 0), (37, 11, 5, 0)])
def test_ns_gemm_ragged(M, N, K, pad):
    _check(M, N, K, pad=pad)


def test_ns_gemm_epilogue_axpby_and_transpose():
    _check(256, 512, 320, alpha=2.0315, beta=-4.7750)
    _check(200, 328, 96, alpha=1.0, beta=3.4445, with_t=True, pad=8)


def test_ns_gemm_quintic_iteration_8b_shape():
    """The three GEMMs of one Newton-Schulz iteration on a normalised
    1024 x 4096 matrix (the Llama-3-8B k_proj), each checked on its own
    inputs: A = W W^T; B = cA A + bA; W' = B W + aW (with W'^T)."""
    a, b, c = 3.4445, -4.7750, 2.0315
    k, L = 1024, 4096
    W = torch.randn(k, L, device="cuda")
    W = (W / W.norm()).to(torch.bfloat16)
    Wt = W.T.contiguous()
    A = torch.empty(k, k, device="cuda", dtype=torch.bfloat16)
    R.ns_gemm_bf16(W, W, A)
    torch.cuda.synchronize()
    ref = W.float() @ W.float().T
    assert ((A.float() - ref).abs() <= 2 ** -8 * ref.abs() + 2 * L * 2 ** -24 * (W.float().abs() @ W.float().abs().T)).all()
    Bm = torch.empty_like(A)
    R.ns_gemm_bf16(A, A, Bm, c, b, A)
    torch.cuda.synchronize()
    ref = c * (A.float() @ A.float().T) + b * A.float()
    mag = abs(c) * (A.float().abs() @ A.float().abs().T) + abs(b) * A.float().abs()
    assert ((Bm.float() - ref).abs() <= 2 ** -8 * ref.abs() + 2 * k * 2 ** -24 * mag).all()
    W2 = torch.empty_like(W)
    W2t = torch.empty_like(Wt)
    R.ns_gemm_bf16(Bm, Wt, W2, 1.0, a, W, W2t)
    torch.cuda.synchronize()
    ref = Bm.float() @ W.float() + a * W.float()
    mag = Bm.float().abs() @ W.float().abs() + abs(a) * W.float().abs()
    assert ((W2.float() - ref).abs() <= 2 ** -8 * ref.abs() + 2 * k * 2 ** -24 * mag).all()
    assert torch.equal(W2t.view(torch.int16), W2.T.contiguous().view(torch.int16))


@pytest.mark.parametrize("M,K,beta", [(128, 64, 0.0), (1024, 4096, 0.0), (1000, 136, 0.0), (24, 40, 0.0),
                                      (1024, 1024, -4.775), (640, 72, 3.0)])
def test_ns_gemm_symmetric(M, K, beta):
    """rsdb_ns_gemm_bf16_sym: W W^T (and c A A + b A with A symmetric):
    upper-triangle tiles + mirror; C exactly symmetric, every element within
    the bound, including the mirrored ones."""
    W = _mat(M, K, _ld(K, 0), 7)
    if beta != 0.0:  # A symmetric operand, D = A
        A0 = (W.float() @ W.float().T / K).to(torch.bfloat16)
        W = A0
        K = M
    C = torch.full((M, _ld(M, 0)), float("nan"), device="cuda", dtype=torch.bfloat16)[:, :M]
    alpha = 2.0315 if beta != 0.0 else 1.0
    R.ns_gemm_bf16_sym(W, W, C, alpha, beta, W if beta != 0.0 else None)
    torch.cuda.synchronize()
    ref = alpha * (W.float() @ W.float().T)
    mag = abs(alpha) * (W.float().abs() @ W.float().abs().T)
    if beta != 0.0:
        ref = ref + beta * W.float()
        mag = mag + abs(beta) * W.float().abs()
    assert torch.isfinite(C.float()).all()
    assert torch.equal(C.view(torch.int16), C.T.contiguous().view(torch.int16))
    err = (C.float() - ref).abs()
    assert (err <= 2.0 ** -8 * ref.abs() + 2 * K * 2.0 ** -24 * mag + 1e-30).all()


def test_ns_gemm_rejects_bad_arguments():
    A = torch.zeros(16, 20, device="cuda", dtype=torch.bfloat16)  # ld 20: not a multiple of 8
    C = torch.zeros(16, 16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(R.RsdbError):
        R.ns_gemm_bf16(A, A, C)
