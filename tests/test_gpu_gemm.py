"""tcgen05 weight-streaming GEMM vs an fp32 torch reference of the same op
(bf16 inputs, fp32 accumulation) and vs the SIMT kernel; row independence
(bitwise) across token-tile sizes, which the greedy spec == regular
invariant relies on."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def handle():
    import paper_2404_15778_b200 as B
    return B.DeviceWeights(B.ModelConfig(1, 2, 128, 64, 256, 64), "bf16")


SHAPES = [(1, 128, 64), (8, 384, 256), (16, 4608, 4608), (17, 13824, 4608), (64, 4608, 18432),
          (100, 640, 768), (256, 1024, 512), (300, 512, 1024), (600, 256, 2048), (33, 50272, 4608)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_tc_gemm_matches_fp32_reference(handle, M, N, K):
    import torch
    from paper_2404_15778_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    ref = x.float() @ w.float().T
    y = handle.gemm(x, w, L.GEMM_TC)
    scale = ref.abs().max().item()
    err = (y - ref).abs().max().item() / scale
    assert err < 1e-4, err
    ys = handle.gemm(x, w, L.GEMM_SIMT)
    assert (ys - ref).abs().max().item() / scale < 1e-4


def test_tc_gemm_rows_bitwise_independent_of_m(handle):
    import torch
    from paper_2404_15778_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(5)
    N, K = 13824, 4608
    x = torch.randn(300, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    full = handle.gemm(x, w, L.GEMM_TC)
    for m in (1, 8, 16, 40, 64, 65, 128, 200, 256):
        part = handle.gemm(x[:m], w, L.GEMM_TC)
        assert torch.equal(part, full[:m]), m


@pytest.mark.parametrize("N,K,M", [(4608, 4608, 1100), (4608, 18432, 1100), (13824, 4608, 1100),
                                   (2048, 8192, 1100), (13824, 4608, 1024)])
def test_serial_split_k_prefill_rows_bitwise_equal_clustered(handle, N, K, M):
    """Prefill-sized M (> 256 rows) runs the serial split-K kernel: one CTA per
    (token group, tile), the S partials accumulated one after another and
    summed in split order — the same bits as the clustered split-K that
    decode / verify blocks use (so prompt rows and later rows agree).  M = 1024
    with two splits takes the 256-token serial tiles."""
    import torch
    from paper_2404_15778_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(N + K)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    full = handle.gemm(x, w, 3)              # packed weights, M > 256: serial split-K
    for lo, hi in ((0, 200), (300, 500), (M - 100, M)):
        part = handle.gemm(x[lo:hi].contiguous(), w, 3)   # M <= 256: clustered split-K
        assert torch.equal(part, full[lo:hi]), (lo, hi)
    ref = x.float() @ w.float().T
    assert (full - ref).abs().max().item() / ref.abs().max().item() < 1e-4
