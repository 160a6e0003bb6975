"""GPU parity of the hand-written tcgen05 int8 GEMM (kernels_imma.cuh) through the C-ABI
(fdfb_gemm_i8, raw int32 epilogue) against exact integer matrix products in numpy.

The GEMM carries both key switches, Shift's VectorPack
and Permute; their end-to-end bytes are checked against the oracle in
test_gpu_parity.py.  Here the contraction itself: ragged M / N / K tails (TMA zero fill and
epilogue masks), several tiles and waves, the int8 extremes, and a long K.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_02731_b200 import Context  # noqa: E402

DEV = torch.device("cuda", 0)
_ctx = {}


def ctx():
    if "c" not in _ctx:
        _ctx["c"] = Context(synth.load_config("tiny"), 0)
    return _ctx["c"]


def ref(A, B):
    return (A.astype(np.int64) @ B.astype(np.int64).T).astype(np.int64)


@pytest.mark.parametrize("M,Nc,K", [(1, 1, 16), (128, 224, 128), (300, 500, 1040), (257, 449, 4096),
                                    (1000, 2300, 272), (64, 224 * 3, 8192 + 16)])
def test_gemm_i8_matches_integer_product(M, Nc, K):
    rng = np.random.default_rng(M * 7 + Nc + K)
    A = rng.integers(-128, 128, (M, K), dtype=np.int8)
    B = rng.integers(-128, 128, (Nc, K), dtype=np.int8)
    D = ctx().gemm_i8(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(D.cpu().numpy().astype(np.int64), ref(A, B))


def test_gemm_i8_extremes_and_many_tiles():
    """All -128 x -128 (the largest positive int32 sums), all -128 x 127, a grid of 160 tiles, and
    one of 6 x 74 + 1 tiles so every persistent CTA (pair) runs >= 6 tiles through both TMEM
    accumulator buffers (each buffer's full/empty barriers through several phases)."""
    K = 2048
    for a, b in ((-128, -128), (-128, 127), (127, 127)):
        A = np.full((130, K), a, np.int8)
        B = np.full((230, K), b, np.int8)
        D = ctx().gemm_i8(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV))
        torch.cuda.synchronize()
        assert (D.cpu().numpy() == a * b * K).all()
    rng = np.random.default_rng(3)
    A = rng.integers(-128, 128, (128 * 20, 512), dtype=np.int8)
    B = rng.integers(-128, 128, (224 * 16, 512), dtype=np.int8)
    D = ctx().gemm_i8(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(D.cpu().numpy().astype(np.int64), ref(A, B))
    # >= 6 tiles per persistent CTA (pair): both TMEM accumulator buffers through several phases
    A = rng.integers(-128, 128, (256, 1024), dtype=np.int8)
    B = rng.integers(-128, 128, (224 * 6 * 74 + 13, 1024), dtype=np.int8)
    D = ctx().gemm_i8(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(D.cpu().numpy().astype(np.int64), ref(A, B))


@pytest.mark.parametrize("M,Nc,K", [(300, 448 * 3, 1040), (257, 448 * 160, 512)])
def test_gemm_i8_wide_tiles(M, Nc, K, monkeypatch):
    """The 448-column pair tiles (two N = 224 MMAs per k-step, one accumulator) that long-K
    contractions (Shift, Permute) use, forced at small K; 160 tiles -> several per pair."""
    monkeypatch.setenv("FDFB_IMMA_WIDE_K", "256")
    c = Context(synth.load_config("tiny"), 0)
    rng = np.random.default_rng(M + Nc + K)
    A = rng.integers(-128, 128, (M, K), dtype=np.int8)
    B = rng.integers(-128, 128, (Nc, K), dtype=np.int8)
    D = c.gemm_i8(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(D.cpu().numpy().astype(np.int64), ref(A, B))
