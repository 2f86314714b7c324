"""Probe: int8 tensor-core GEMM throughput on this GPU for the key-switch-as-GEMM shape
(M gates x K = N1*t*3 one-hot selector columns x N = 4 byte planes * (n+1))."""
import time, torch
for M in (140, 544, 4096):
    K, N = 1024 * 8 * 3, 4 * 631
    N = (N + 15) // 16 * 16
    a = torch.randint(0, 2, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (K, N), dtype=torch.int8, device="cuda")
    Mp = max(M, 32)
    if Mp != M:
        a = torch.nn.functional.pad(a, (0, 0, 0, Mp - M))
    c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"M={M} K={K} N={N}: {ms:.4f} ms, {2*Mp*K*N/ms/1e9:.1f} TOPS")
