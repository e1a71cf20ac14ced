import torch, time, numpy as np
n = 1 << 28  # 2 GiB of f64
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, src in (("torch pinned", h), ("from_numpy(pinned view)", torch.from_numpy(h.numpy()))):
    print(name, "is_pinned", src.is_pinned())
    for _ in range(2): d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(3): d.copy_(src, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(name, "H2D GB/s", 3 * n * 8 / e0.elapsed_time(e1) / 1e6)
e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H GB/s", n * 8 / e0.elapsed_time(e1) / 1e6)
# split into 4 concurrent streams
ss = [torch.cuda.Stream() for _ in range(4)]
torch.cuda.synchronize(); e0.record()
q = n // 4
for i, s in enumerate(ss):
    with torch.cuda.stream(s):
        d[i*q:(i+1)*q].copy_(h[i*q:(i+1)*q], non_blocking=True)
for s in ss: torch.cuda.current_stream().wait_stream(s)
e1.record(); torch.cuda.synchronize()
print("H2D 4 streams GB/s", n * 8 / e0.elapsed_time(e1) / 1e6)
import subprocess; print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
