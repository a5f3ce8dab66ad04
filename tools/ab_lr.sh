mkdir -p gpurun_out
for r in 1 2; do for n in base u2 u8 u8b4; do
 PV_LIB_PATH=$PWD/build_ab/libpovar_$n.so timeout 300 python tools/time_terms.py vlarge 2>&1 | tail -2
 PV_LIB_PATH=$PWD/build_ab/libpovar_$n.so timeout 300 python tools/lm_iter_time.py vlarge 10 2>&1 | tail -1
done; done
