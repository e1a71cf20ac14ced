set -x
python tools/kbench.py --cases c5shard,c5shard_t --reps 12 2>&1 | grep c5shard | head -2
HSK_SJLT_RPT=1 python tools/kbench.py --cases c5shard --reps 12 2>&1 | grep '"c5shard' | head -1
HSK_SJLT_STAGES=2 python tools/kbench.py --cases c5shard --reps 12 2>&1 | grep '"c5shard' | head -1
HSK_SJLT_TK=64 python tools/kbench.py --cases c5shard --reps 12 2>&1 | grep '"c5shard' | head -1
HSK_NVCC_EXTRA="-DHSK_SJLT_MULTICAST=1 -DHSK_TUNING=1" python -m paper_2302_01977_b200.build --force > /dev/null 2>&1
for mc in 2 4 8; do HSK_SJLT_MC=$mc timeout 120 python tools/kbench.py --cases c5shard,c5shard_t --reps 12 2>&1 | grep '"c5shard' | head -2; done
HSK_SJLT_W32=1 timeout 120 python tools/kbench.py --cases c5shard,c5shard_t --reps 12 2>&1 | grep '"c5shard' | head -2
