# Gaussian split-K A/B (HSK_GAUSS_SPLITS) on C2 and the C5 row shard shape
for sp in 1 2 3 4 5; do HSK_GAUSS_SPLITS=$sp python tools/kbench.py --cases c2g --reps 20 2>&1 | grep '"env"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())['results']; print($sp, {k: round(v['ms'],3) for k,v in d.items()})"; done
