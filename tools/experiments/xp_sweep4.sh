# S' on 128-row tiles (d <= 64): XOR-layout transposing producers (mode 4) vs the
# S-layout staging ring (mode 5, HSK_SJLT_XP=1): chunk size x staging group sweep
mkdir -p gpurun_out
for cfg in "off:HSK_SJLT_XP=0" "64x2:HSK_SJLT_XP=1" "64x1:HSK_SJLT_XP=1 HSK_SJLT_XP_GB=1" "64x4:HSK_SJLT_XP=1 HSK_SJLT_XP_GB=4" "48x3:HSK_SJLT_XP=1 HSK_SJLT_TK_T=48 HSK_SJLT_XP_GB=3" "48x1:HSK_SJLT_XP=1 HSK_SJLT_TK_T=48 HSK_SJLT_XP_GB=1" "32x2:HSK_SJLT_XP=1 HSK_SJLT_TK_T=32 HSK_SJLT_XP_GB=2" "32x1:HSK_SJLT_XP=1 HSK_SJLT_TK_T=32 HSK_SJLT_XP_GB=1" "80x5:HSK_SJLT_XP=1 HSK_SJLT_TK_T=80 HSK_SJLT_XP_GB=5"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "$name $(env $envs timeout 600 python tools/kbench.py --cases ${CASES:-sj-16384-64-4,sj-16384-64-2,sj-16384-32-4,c3a4} --reps 20 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],4) for k,v in d.items() if k.endswith('St')})")"
done
