for v in libhprop_b200.so libhprop_b200_smemw.so libhprop_b200.so libhprop_b200_smemw.so; do
echo $v; HP_LIB_VARIANT=$v timeout 120 python tools/time_matvec.py cfg4 20
done
for v in libhprop_b200.so libhprop_b200_smemw.so; do
HP_LIB_VARIANT=$v timeout 300 python tools/bench_propagate.py cfg4 --steps 5 --cpu-steps 0 2>&1 | tail -1
done
HP_FG_QUAD=0 timeout 300 python tools/bench_propagate.py cfg4 --steps 5 --cpu-steps 0 2>&1 | tail -1
