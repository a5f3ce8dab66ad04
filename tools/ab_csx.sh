# A/B of two builds on the stage-1 LM iteration and per-operation times (vlarge)
mkdir -p gpurun_out
for r in 1 2; do for n in ${AB_VARIANTS:-base csx}; do
 PV_LIB_PATH=$PWD/build_ab/libpovar_$n.so timeout 300 python tools/time_ops.py vlarge 5 2>&1 | tail -8
 PV_LIB_PATH=$PWD/build_ab/libpovar_$n.so timeout 300 python tools/lm_iter_time.py vlarge 10 2>&1 | tail -1
done; done
