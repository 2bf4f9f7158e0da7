"""cuBLAS FP64 reference rates (DGEMM / ZGEMM via torch.matmul) on the B200 box."""
import torch, time
def rate(dtype, n, flop_per_mac, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda"); b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flop_per_mac * n**3 / best / 1e9, best
print("DGEMM 8192: %.2f TFLOP/s (%.2f ms)" % rate(torch.float64, 8192, 2))
print("ZGEMM 4096: %.2f TFLOP/s (%.2f ms)" % rate(torch.complex128, 4096, 8))
print("ZGEMM 8192: %.2f TFLOP/s (%.2f ms)" % rate(torch.complex128, 8192, 8, reps=4))
