# TK / stages / L2-prefetch sweep of the SJLT kernels (one process per setting):
#   CASES=c2s,c5shard bash tools/experiments/tk_sweep.sh <tag> "TK:STAGES:PF ..."
tag=$1; shift
mkdir -p gpurun_out
for cfg in $1; do
  IFS=: read tk stg pf <<< "$cfg"
  env ${tk:+HSK_SJLT_TK=$tk} ${tk:+HSK_SJLT_TK_T=$tk} ${stg:+HSK_SJLT_STAGES=$stg} ${pf:+HSK_SJLT_PF=$pf} \
    timeout 600 python tools/kbench.py --cases ${CASES:-c2s} --reps 30 > gpurun_out/tk_${tag}_$cfg.json 2>&1
  echo "== $cfg $(tail -1 gpurun_out/tk_${tag}_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print(' '.join(f'{k}={v[\"ms\"]:.4f}' for k,v in d.items()))")"
done
