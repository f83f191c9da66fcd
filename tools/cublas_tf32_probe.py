"""cuBLAS TF32 at 4096^3 in two operand layouts (development probe):
  tt: torch.mm(a.t(), b.t()) - what measure.py timed (cuBLAS sees both
      operands K-major, kernel ..._ttn_...)
  nn: torch.mm(bT, aT) with contiguous bT (N,K) and aT (K,M): memory of the
      result is C column-major = A (col-major M x K) x B (col-major K x N),
      exactly the problem the sgemm_tc kernels solve (A MN-major)."""
import torch

torch.backends.cuda.matmul.allow_tf32 = True
M = N = K = 4096
R = 3
aa = [torch.randn(K, M, device="cuda") for _ in range(R)]   # A col-major storage = (K, M) row-major
bb = [torch.randn(N, K, device="cuda") for _ in range(R)]   # B col-major storage = (N, K) row-major


def t(fn, reps=30):
    for i in range(3):
        fn(i % R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for i in range(reps):
            fn(i % R)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


tt = t(lambda i: torch.mm(aa[i].t(), bb[i].t()))
nn = t(lambda i: torch.mm(bb[i], aa[i]))
print(f"cublas tf32 4096^3: tt (both K-major) {tt:.1f} us   nn (A MN-major, our layout) {nn:.1f} us")
