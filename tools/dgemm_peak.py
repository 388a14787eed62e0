"""cuBLAS DGEMM throughput (torch.matmul float64) — FP64 roofline yardstick."""
import torch, time, json
res = {}
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n**3 / (best * 1e-3) / 1e12
    print(f"dgemm n={n}: {res[n]:.2f} TFLOP/s ({best:.2f} ms)")
# sustained
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4:
    c = a @ b; cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"dgemm sustained n=8192: {2*n**3*cnt/(e0.elapsed_time(e1)*1e-3)/1e12:.2f} TFLOP/s")
# batched small: 16384 x 64x64
for (bs, m) in ((16384, 64), (1024, 368), (64, 1520)):
    a = torch.randn(bs, m, m, dtype=torch.float64, device="cuda"); b = torch.randn(bs, m, m, dtype=torch.float64, device="cuda")
    for _ in range(3): c = torch.bmm(a, b)
    torch.cuda.synchronize(); e0.record(); c = torch.bmm(a, b); e1.record(); torch.cuda.synchronize()
    print(f"bmm {bs}x{m}^3: {2*bs*m**3/(e0.elapsed_time(e1)*1e-3)/1e12:.2f} TFLOP/s")
# copy bandwidth
x = torch.empty(2**30 // 8 * 4, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
print(f"copy: {2*x.numel()*8/(e0.elapsed_time(e1)*1e-3)/1e9:.1f} GB/s")
