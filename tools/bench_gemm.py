"""Microbenchmark of the library's tcgen05 GEMM (climber_debug_gemm) on the
hot path's shapes: TFLOP/s from CUDA events."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_09888_b200.climber import debug_gemm

shapes = [(65536, 1536, 512), (65536, 512, 512), (65536, 2048, 512), (65536, 512, 2048), (65536, 1024, 4096),
          (65536, 4096, 1024), (32768, 1536, 512)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in sys.argv[1].split(","))]
reps = int(os.environ.get("REPS", "20"))
EPI = int(os.environ.get("EPI", "0"))
for M, N, K in shapes:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    D = torch.zeros(M, N, device="cuda") if EPI == 0 else torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        debug_gemm(A, B, D, epi=EPI)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        debug_gemm(A, B, D, epi=EPI)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        torch.matmul(A, B.T)
    t1.record()
    torch.cuda.synchronize()
    ms_t = t0.elapsed_time(t1) / reps
    print(json.dumps({"epi": EPI, "M": M, "N": N, "K": K, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9,
                      "torch_bf16_out_tflops": 2 * M * N * K / ms_t / 1e9}), flush=True)
