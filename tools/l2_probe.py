"""L2 residency probe: warm bandwidth of plain torch copies vs working-set size."""
import torch
dev = torch.device("cuda:0")
for mb in (8, 32, 64, 96, 128, 256, 1024):
    n = mb * (1 << 20) // 8
    a = torch.randn(n, dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record(s)
    for _ in range(reps):
        b.copy_(a)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"copy {mb:5d} MB (x2 traffic): {ms*1e3:8.1f} us  {2*mb*(1<<20)/ms/1e6:8.0f} GB/s", flush=True)
