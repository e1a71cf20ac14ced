timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for lib in "" "_exp/ab/libhsk_prev.so"; do echo "lib=$lib"; HSK_LIB=$lib timeout 300 python tools/kbench.py --cases c1,c2s,c3,c5s 2>&1 | grep -v env | cut -c1-240; done
