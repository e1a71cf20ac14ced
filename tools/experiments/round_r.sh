# round r02r: tests, bench, launch list, ncu of the headline kernel and the transposed-tile S' kernels
set -x
tag=r02r
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_all_$tag.log 2>&1; tail -3 gpurun_out/pt_all_$tag.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ncu_l_$tag.log 2>&1; echo ncu_list=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sjlt_apply -s 5 -c 1 \
  -o gpurun_out/prof_bench_sjlt_$tag -f python bench.py --steps 2 --warmup 5 --no-configs --no-cpu > gpurun_out/ncu_f_$tag.log 2>&1; echo ncu_bench=$?
for c in xp8_St xp4_St c3a4_St; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sjlt_apply -s 1 -c 1 \
    -o gpurun_out/prof_${c}_$tag -f python tools/prof_once.py $c > gpurun_out/ncu_${c}_$tag.log 2>&1; echo ncu_$c=$?
done
ls -la gpurun_out | tail -20; du -sh gpurun_out
