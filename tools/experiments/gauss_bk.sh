# Gaussian DMMA GEMM A/B: BK, stages, min resident CTAs (register cap)
for cfg in "16 2 1" "16 2 4" "16 2 5" "16 3 5"; do set -- $cfg
  HSK_NVCC_EXTRA="-DHSK_GAUSS_BK=$1 -DHSK_GAUSS_STAGES=$2 -DHSK_GAUSS_MINB=$3" python -m paper_2302_01977_b200.build --force > /dev/null 2>&1 || { echo "build failed"; continue; }
  echo "BK=$1 stages=$2 minb=$3 $(python tools/kbench.py --cases c2g --reps 20 2>&1 | grep '"env"' | python -c "import json,sys; d=json.loads(sys.stdin.read())['results']; print({k: round(v['ms'],3) for k,v in d.items()})")"
done
