set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_all_r02q.log 2>&1; tail -3 gpurun_out/pt_all_r02q.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02q.json 2> gpurun_out/bench_r02q.err; echo bench=$?
timeout 1500 python tools/paper_table.py --out gpurun_out/paper_table71_r02q.json > gpurun_out/paper_table_r02q.log 2>&1; echo table=$?
HSK_SJLT_XP=0 timeout 1500 python tools/paper_table.py --out gpurun_out/paper_table71_r02q_xp0.json > gpurun_out/paper_table_r02q_xp0.log 2>&1; echo table0=$?
