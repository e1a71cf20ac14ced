import ctypes
import itertools
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "stream_probe.so"))
lib.probe_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64] + [ctypes.c_int] * 6 + [ctypes.c_void_p, ctypes.c_void_p]
n = 16384
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
sink = torch.zeros(4096, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def run(br, bc, stages, nslabs, pers, grid=0, reps=10):
    f = lambda: lib.probe_run(A.data_ptr(), n, n, br, bc, stages, nslabs, pers, grid, sink.data_ptr(), st)
    for _ in range(2):
        assert f() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return n * n * 8 / ms / 1e6


for (br, bc) in [(32, 256), (64, 128), (128, 64), (256, 32), (64, 64), (128, 128), (256, 64)]:
    box = br * bc * 8
    for stages in (2, 3, 4, 6, 8):
        if 1024 + stages * box > 227 * 1024:
            continue
        res = []
        for nslabs, pers in ((1, 0), (2, 0), (1, 1), (2, 1)):
            res.append(f"s{nslabs}p{pers}={run(br, bc, stages, nslabs, pers):.0f}")
        print(f"box {br}x{bc} ({box//1024}KB) stages {stages}: " + " ".join(res), flush=True)
