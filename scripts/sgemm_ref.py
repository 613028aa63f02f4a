"""cuBLAS FP32 (no TF32) SGEMM throughput on this GPU: the practical FFMA GEMM
ceiling the fused FFMA kernels are compared with."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
for (m, n, k) in [(8192, 8192, 8192), (16384, 512, 64), (65536, 128, 64), (4096, 4096, 4096)]:
    a = torch.randn(m, k, device="cuda")
    b = torch.randn(k, n, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    s.record()
    for _ in range(it):
        c = a @ b
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / it
    print(f"sgemm {m}x{n}x{k}: {2 * m * n * k / ms / 1e9:.1f} TFLOP/s ({ms:.3f} ms)")
