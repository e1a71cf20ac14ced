# S' on tiles transposed in shared memory (modes 5 / 6): chunk size x staging group sweep
mkdir -p gpurun_out
for cfg in "off:HSK_SJLT_XP=0" "128x8:HSK_SJLT_XP_GB=8" "128x4:HSK_SJLT_XP_GB=4" "128x2:HSK_SJLT_XP_GB=2" "96x6:HSK_SJLT_TK_T=96 HSK_SJLT_XP_GB=6" "96x3:HSK_SJLT_TK_T=96 HSK_SJLT_XP_GB=3" "96x2:HSK_SJLT_TK_T=96 HSK_SJLT_XP_GB=2" "64x4:HSK_SJLT_TK_T=64 HSK_SJLT_XP_GB=4" "64x2:HSK_SJLT_TK_T=64 HSK_SJLT_XP_GB=2" "80x5:HSK_SJLT_TK_T=80 HSK_SJLT_XP_GB=5" "112x7:HSK_SJLT_TK_T=112 HSK_SJLT_XP_GB=7"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "$name $(env $envs timeout 600 python tools/kbench.py --cases ${CASES:-c1,sj-16384-128-4,sj-16384-256-8,c3} --reps 20 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],4) for k,v in d.items() if k.endswith('St')})")"
done
