# A/B of SJLT kernel builds on one box: bash tools/experiments/ab_r02d.sh <tag> <lib names...>
# (libs under _exp/ab/libhsk_<name>.so; "new" = the in-tree build)
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -x -q > gpurun_out/pt_$tag.log 2>&1; tail -2 gpurun_out/pt_$tag.log
for lib in "$@"; do
  if [ $lib = new ]; then L=""; else L=_exp/ab/libhsk_$lib.so; fi
  HSK_LIB=$L timeout 600 python tools/kbench.py --cases ${CASES:-c1,c2s,c5shard,c5shard_t,c3} --reps 20 > gpurun_out/kb_${tag}_$lib.json 2>&1
  echo "== $lib"; tail -1 gpurun_out/kb_${tag}_$lib.json | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print(' '.join(f'{k}={v[\"ms\"]:.4f}' for k,v in d.items()))"
done
