"""cuBLAS bf16 GEMM times for the implicit-GEMM shapes of the convolutions (reference
for the conv kernels' per-tile efficiency; CUDA events, 20 reps after warm-up)."""
import torch
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
for (M, K, N) in [(131072, 576, 64), (65536, 576, 64), (131072, 64, 256), (200704, 576, 64), (50176, 1152, 128),
                  (12544, 2304, 256), (200704, 64, 256), (200704, 256, 64)]:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"M={M} K={K} N={N}: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TFLOP/s  {(M*K+K*N+M*N)*2/ms/1e6:.0f} GB/s", flush=True)
