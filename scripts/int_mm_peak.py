"""cuBLASLt int8 GEMM (torch._int_mm) throughput at 8192^3: the library-achievable int8 yardstick."""
import torch, json
a = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
for _ in range(3): torch._int_mm(a, b.t())
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): c = torch._int_mm(a, b.t())
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(json.dumps({"torch._int_mm_8192": True, "ms": ms, "tops": 2 * 8192**3 / (ms * 1e-3) / 1e12}))
