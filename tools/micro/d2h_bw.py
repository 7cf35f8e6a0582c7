"""Dev probe: host<->device copy bandwidth for the S24 output size (pred pad32 + level)."""
import torch, time
n = 1 << 24
for nbytes in (n * 8, n * 4):
    d = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
    h = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
    s = torch.cuda.Stream()
    for _ in range(3):
        h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(10): h.copy_(d, non_blocking=True)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"D2H {nbytes/1e6:.0f} MB: {ms:.3f} ms = {nbytes/ms/1e6:.1f} GB/s")
    a.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"H2D {nbytes/1e6:.0f} MB: {ms:.3f} ms = {nbytes/ms/1e6:.1f} GB/s")
