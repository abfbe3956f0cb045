"""Host-side f32 <-> bf16 conversion throughput vs PCIe copy bandwidth on the GPU box (decides
where the float host-buffer path converts)."""
import time

import torch

torch.set_num_threads(16)
n = 1 << 28  # 1 GiB of float32
x = torch.rand(n, dtype=torch.float32).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16).pin_memory()
for _ in range(2):
    y.copy_(x)
t = time.perf_counter()
for _ in range(5):
    y.copy_(x)
dt = (time.perf_counter() - t) / 5
print(f"host f32->bf16 copy_: {n * 6 / dt / 1e9:.1f} GB/s moved ({n * 4 / dt / 1e9:.1f} GB/s of f32 read), {dt*1e3:.1f} ms per GiB f32")
z = torch.empty(n, dtype=torch.float32).pin_memory()
t = time.perf_counter()
for _ in range(5):
    z.copy_(y)
dt = (time.perf_counter() - t) / 5
print(f"host bf16->f32 copy_: {dt*1e3:.1f} ms per GiB f32 out")
t = time.perf_counter()
ok = torch.isfinite(x).all().item()
print(f"isfinite over 1 GiB f32: {(time.perf_counter() - t)*1e3:.1f} ms")
d = torch.empty(n, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"H2D pinned: {n * 4 / dt / 1e9:.1f} GB/s")
t = time.perf_counter()
for _ in range(3):
    x.copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"D2H pinned: {n * 4 / dt / 1e9:.1f} GB/s")
