for w in 1000 0 100 300; do HSK_SJLT_WAIT_NS=$w python tools/kbench.py --cases c2s,c3,c1 --reps 40 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($w, {k: round(v['ms'],4) for k,v in d['results'].items()})"; done
