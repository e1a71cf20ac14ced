# C2 S: warp shape x TK (production lib): HSK_SJLT_W32 / HSK_SJLT_TK
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -x -q 2>&1 | tail -1
for cfg in "0:0" "24:128" "24:96" "20:96" "20:112" "16:128"; do
  IFS=: read w tk <<< "$cfg"
  env HSK_SJLT_W32=$w HSK_SJLT_TK=$tk timeout 600 python tools/kbench.py --cases c2s,c1 --reps 40 > gpurun_out/kb_st_$w_$tk.json 2>&1
  echo "== W$w TK$tk $(tail -1 gpurun_out/kb_st_$w_$tk.json | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print(' '.join(f'{k}={v[\"ms\"]:.4f}' for k,v in d.items()))")"
done
