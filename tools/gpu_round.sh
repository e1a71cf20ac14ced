# One GPU round: full gpu tests, kernel bench, bench.py, ncu launch list and
# one full capture of the bench's SJLT kernel (each ncu only after the same
# command exited 0 without ncu).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
timeout 400 python tools/kbench.py --cases c1,c2s,c2g,c3,c4,c5s 2>&1 | grep -v env > gpurun_out/kb.log; cat gpurun_out/kb.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$?; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --steps 2 --warmup 3 > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_l.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sjlt_apply -s 4 -c 1 -o gpurun_out/prof_bench_sjlt -f python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_f.log 2>&1; echo ncu2=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload c5_rowshard --steps 5 --warmup 3 > gpurun_out/rowshard.log 2>&1; echo rowshard=$?; tail -1 gpurun_out/rowshard.log
