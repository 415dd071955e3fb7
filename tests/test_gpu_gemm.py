"""The tcgen05 bf16 GEMM in isolation vs a plain fp64 matmul of the same
bf16 operands (fp32 accumulation: tolerance from K * 2^-24 * |a||b|)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 256, 512), (1000, 1536, 512), (4096, 512, 2048),
                                   (77, 384, 128), (2048, 1024, 4096), (129, 128, 192)])
@pytest.mark.parametrize("use_tc", [True, False])
def test_gemm_vs_fp64(M, N, K, use_tc):
    import torch
    from paper_2502_09888_b200.climber import debug_gemm
    g = torch.Generator().manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    D0 = torch.randn(M, N, generator=g)
    D = D0.clone().cuda()
    debug_gemm(A.cuda(), B.cuda(), D, use_tc=use_tc)
    torch.cuda.synchronize()
    ref = D0.double() + A.double() @ B.double().T
    err = (D.cpu().double() - ref).abs().max().item()
    bound = K * 2.0 ** -22 * 16  # |a|,|b| ~ N(0,1): generous fp32-accumulation bound
    assert err < bound, (err, bound)


@pytest.mark.parametrize("epi", [1, 2])
@pytest.mark.parametrize("M,N,K", [(300, 256, 512), (4096, 2048, 512), (77, 384, 128)])
def test_gemm_store_epilogues(M, N, K, epi):
    import torch
    import torch.nn.functional as F
    from paper_2502_09888_b200.climber import debug_gemm
    g = torch.Generator().manual_seed(M + N + K + epi)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = (torch.randn(N, K, generator=g) / K ** 0.5).bfloat16()
    D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    debug_gemm(A.cuda(), B.cuda(), D, epi=epi)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T
    if epi == 2:
        ref = F.silu(ref)
    err = (D.cpu().double() - ref).abs().max().item()
    assert err < 2e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K", [(1000, 512, 512), (300, 256, 128)])
def test_gemm_grouped_interleaved(M, N, K):
    """Two GEMMs in one launch over an interleaved [M][2][K] A (the N_b block
    slots of candidate rows): D[:, b] += A[:, b] @ B[b]^T."""
    import torch
    from paper_2502_09888_b200.climber import debug_gemm
    g = torch.Generator().manual_seed(M + N)
    A = torch.randn(M, 2, K, generator=g).bfloat16()
    B = torch.randn(2, N, K, generator=g).bfloat16()
    D0 = torch.randn(M, 2, N, generator=g)
    D = D0.clone().cuda()
    debug_gemm(A.cuda().view(M, 2 * K), B.cuda().view(2 * N, K), D, epi=3)
    torch.cuda.synchronize()
    ref = D0.double().clone()
    for b in range(2):
        ref[:, b] += A[:, b].double() @ B[b].double().T
    err = (D.cpu().double() - ref).abs().max().item()
    assert err < K * 2.0 ** -22 * 16, err
