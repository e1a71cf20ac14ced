"""Per-launch time of the C2 SJLT S kernel vs run length, with power/clock samples."""
import os, subprocess, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import device, matgen
from paper_2302_01977_b200 import sketching as sk
n, d = 16384, int(os.environ.get("SUS_D", "512"))
A = matgen.gaussian_kernel(n, 8, 0.5)
op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=4, construction="block")
S = device.DeviceMatrix.empty(n, d)
blk = op.blocks[0]
f = lambda: device.apply_block(blk, A, False, S, 0)
for _ in range(5): f()
torch.cuda.synchronize()
samples = []
stop = False
def sampler():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        samples.append(out); time.sleep(0.05)
th = threading.Thread(target=sampler); th.start()
for reps in (20, 2000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    print(reps, "reps: ms/launch", round(e0.elapsed_time(e1) / reps, 4), flush=True)
stop = True; th.join()
print("samples (sm MHz, W):", samples[::max(1, len(samples)//12)])
