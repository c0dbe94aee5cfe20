"""Reference rates on this B200: cuBLASLt int8 (torch._int_mm) and bf16 (torch.mm), CUDA events,
best of N.  Context for the KB2 roofline denominator (not part of the product path)."""
import json
import torch

def bench(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best

out = {}
for (m, n, k) in [(8192, 8192, 8192), (16384, 16384, 16384), (65536, 16384, 10112)]:
    a = torch.randint(0, 2, (m, k), dtype=torch.int8, device="cuda")
    b = torch.randint(0, 2, (n, k), dtype=torch.int8, device="cuda").t()
    ms = bench(lambda: torch._int_mm(a, b))
    out[f"int8_{m}x{n}x{k}_tops"] = 2 * m * n * k / ms / 1e9
    del a, b
    torch.cuda.empty_cache()
a = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
ms = bench(lambda: a @ b)
out["bf16_8192_tflops"] = 2 * 8192**3 / ms / 1e9
print(json.dumps(out))
