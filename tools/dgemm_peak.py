import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"cuBLAS DGEMM {n}^3: {ms:.2f} ms = {2*n**3/ms/1e9:.1f} TFLOP/s")
# C5 shape: K^T (16384x4096) @ R (4096x128)
K = torch.randn(4096, 16384, dtype=torch.float64, device="cuda"); R = torch.randn(4096, 128, dtype=torch.float64, device="cuda"); D = torch.randn(16384, 128, dtype=torch.float64, device="cuda")
for _ in range(3): G = K.t() @ R; Y = K @ D
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): G = K.t() @ R; Y = K @ D
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"C5 pair (K^T R + K D, B=128): {ms:.3f} ms = {4*4096*16384*128/ms/1e9:.1f} TFLOP/s")
