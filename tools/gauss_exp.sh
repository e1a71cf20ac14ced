for sp in 1 2 3 4 5 6 8; do HSK_GAUSS_SPLITS=$sp python tools/kbench.py --cases c2g --reps 20 2>&1 | grep '"c2g_S' ; done
python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2302_01977_b200 import _lib
L = _lib.load()
x = torch.zeros(1, dtype=torch.float64, device='cuda')
for it in (2000, 20000):
    _lib.call("hsk_dmma_probe", it, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _lib.call("hsk_dmma_probe", it, x.data_ptr(), torch.cuda.current_stream().cuda_stream); e1.record(); torch.cuda.synchronize()
    print("dmma probe", it, L.hsk_dmma_probe_flops(it) / e0.elapsed_time(e1) / 1e9, "TF/s")
PY
