# C2 SJLT S / S' TK sweep (the stage count follows from the 226 KB ring budget)
for tk in 208 176 144 136 128 112; do
  HSK_SJLT_TK=$tk HSK_SJLT_TK_T=$tk python tools/kbench.py --cases c2s --reps 40 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print($tk, {k: round(v['ms'],4) for k,v in d.items()})"
done
