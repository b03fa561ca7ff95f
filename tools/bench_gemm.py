"""Per-launch time of the tall-skinny f32 GEMM entry (kifmm_gemm_f32) at the
config-2 operator shapes, back-to-back launches timed with CUDA events."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import _native as nat

dev = torch.device("cuda")
s = torch.cuda.current_stream().cuda_stream
for (M, N, K, asum) in [(32768, 56, 56, 1), (32768, 56, 51, 1), (32768, 51, 56, 1), (4096, 448, 56, 1),
                        (32768, 56, 51, 4), (262144, 56, 56, 1), (32768, 152, 147, 1)]:
    A = torch.randn(M * K * asum, device=dev)
    B = torch.randn(K * N, device=dev)
    C = torch.zeros(M * N, device=dev)
    args = lambda: (M, N, K, 1.0, A.data_ptr(), K * asum, asum, K, B.data_ptr(), N, None,
                    C.data_ptr(), N, None, 0, s)
    for _ in range(3):
        nat.call("kifmm_gemm_f32", *args())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        nat.call("kifmm_gemm_f32", *args())
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    byts = 4.0 * (M * K * asum + M * N + K * N)
    print(f"M={M} N={N} K={K} asum={asum}: {us:7.1f} us  {2.0*M*N*K/us/1e6:6.1f} TF/s  {byts/us/1e3:6.0f} GB/s", flush=True)
