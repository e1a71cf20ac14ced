# C1 (n = 4096, d = 256, alpha = 4 graph): schedule / tile / TK variants on the tuning lib
mkdir -p gpurun_out
for cfg in "base:" "rpt1:HSK_SJLT_RPT=1 HSK_SJLT_RPT_T=1" "sk1:HSK_SJLT_STREAMK=1" "tk64:HSK_SJLT_TK=64 HSK_SJLT_TK_T=64" "tk96:HSK_SJLT_TK=96 HSK_SJLT_TK_T=96" "w16:HSK_SJLT_W32=16" "w24:HSK_SJLT_W32=24" "st2:HSK_SJLT_STAGES=2" "st4:HSK_SJLT_STAGES=4 HSK_SJLT_TK=64 HSK_SJLT_TK_T=64"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env HSK_LIB=_exp/ab/libhsk_tune.so $envs timeout 300 python tools/kbench.py --cases c1 --reps 50 > gpurun_out/kb_c1_$name.json 2>&1
  echo "== $name $(tail -1 gpurun_out/kb_c1_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print(' '.join(f'{k}={v[\"ms\"]*1000:.1f}us' for k,v in d.items()))" 2>&1 | tail -1)"
done
