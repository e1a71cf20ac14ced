# consumer warp-shape A/B (tuning lib, HSK_SJLT_W32 = shape) + the production lib's parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
for w in prod 16 20 23 24; do
  if [ $w = prod ]; then L=""; W=""; else L=_exp/ab/libhsk_tune.so; W=$w; fi
  HSK_LIB=$L HSK_SJLT_W32=$W timeout 600 python tools/kbench.py --cases ${CASES:-c1,c2s,c5shard} --reps 30 > gpurun_out/kb_ws$w.json 2>&1
  echo "== W$w $(tail -1 gpurun_out/kb_ws$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print(' '.join(f'{k}={v[\"ms\"]:.4f}' for k,v in d.items()))")"
done
