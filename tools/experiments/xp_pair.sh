# paired C3 plan: S at TK 128 (is the walker the limit?) and S' on transposed tiles at larger chunks
for cfg in "base:" "S_tk128:HSK_SJLT_TK=128" "S_tk160:HSK_SJLT_TK=160" "xp128x4:HSK_SJLT_XP=1" "xp144x3:HSK_SJLT_XP=1 HSK_SJLT_TK_T=144 HSK_SJLT_XP_GB=3" "xp160x5:HSK_SJLT_XP=1 HSK_SJLT_TK_T=160 HSK_SJLT_XP_GB=5" "xp160x2:HSK_SJLT_XP=1 HSK_SJLT_TK_T=160 HSK_SJLT_XP_GB=2" "xp176x1:HSK_SJLT_XP=1 HSK_SJLT_TK_T=176 HSK_SJLT_XP_GB=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "$name $(env $envs timeout 600 python tools/kbench.py --cases c3 --reps 20 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],4) for k,v in d.items()})")"
done
