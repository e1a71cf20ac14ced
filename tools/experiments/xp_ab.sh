set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_sketch.py -m gpu -x -q > gpurun_out/xp_tests.log 2>&1; tail -5 gpurun_out/xp_tests.log
for xp in 0 -1; do
  if [ $xp = -1 ]; then E=""; else E="HSK_SJLT_XP=$xp"; fi
  env $E timeout 600 python tools/kbench.py --cases c1,sj-16384-128-4,sj-16384-256-4,sj-16384-256-8,c3,c3a4 --reps 20 2>&1 | grep -v '"env"' | tee -a gpurun_out/xp_ab_$xp.log
done
