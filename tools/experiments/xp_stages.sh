# transposed S' tiles: more, smaller ring slots (HSK_SJLT_STAGES) at smaller chunks
for cfg in "128x4s2:" "96x3s3:HSK_SJLT_TK_T=96 HSK_SJLT_XP_GB=3 HSK_SJLT_STAGES=3" "96x2s3:HSK_SJLT_TK_T=96 HSK_SJLT_XP_GB=2 HSK_SJLT_STAGES=3" "80x5s3:HSK_SJLT_TK_T=80 HSK_SJLT_XP_GB=5 HSK_SJLT_STAGES=3" "64x4s4:HSK_SJLT_TK_T=64 HSK_SJLT_XP_GB=4 HSK_SJLT_STAGES=4" "64x4s3:HSK_SJLT_TK_T=64 HSK_SJLT_XP_GB=4 HSK_SJLT_STAGES=3" "64x2s4:HSK_SJLT_TK_T=64 HSK_SJLT_XP_GB=2 HSK_SJLT_STAGES=4" "112x7s2:HSK_SJLT_TK_T=112 HSK_SJLT_XP_GB=7"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "$name $(env $envs timeout 600 python tools/kbench.py --cases sj-16384-128-4,sj-16384-256-8,sj-16384-192-8 --reps 20 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],4) for k,v in d.items() if k.endswith('St')})")"
done
for cfg in "64x2s2:" "32x2s3:HSK_SJLT_TK_T=32 HSK_SJLT_XP_GB=2 HSK_SJLT_STAGES=3" "32x2s4:HSK_SJLT_TK_T=32 HSK_SJLT_XP_GB=2 HSK_SJLT_STAGES=4" "48x3s3:HSK_SJLT_TK_T=48 HSK_SJLT_XP_GB=3 HSK_SJLT_STAGES=3" "32x1s4:HSK_SJLT_TK_T=32 HSK_SJLT_XP_GB=1 HSK_SJLT_STAGES=4"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "rpt4 $name $(env $envs timeout 600 python tools/kbench.py --cases sj-16384-64-4,sj-16384-64-2,c3a4 --reps 20 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],4) for k,v in d.items() if k.endswith('St')})")"
done
