import torch, time
def tm(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for B, m, n in [(1, 256, 128), (64, 256, 128), (64, 256, 64), (128, 256, 128), (1, 256, 64), (1, 64, 64)]:
    X = torch.randn(B, m, n, dtype=torch.float64, device="cuda")
    print(B, m, n, "qr %.3f ms" % tm(lambda: torch.linalg.qr(X, mode="reduced")),
          "geqrf %.3f ms" % tm(lambda: torch.geqrf(X)))
