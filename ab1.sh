mkdir -p gpurun_out/ab1
A=paper_1711_10413_b200/_build/ab/libA.so
B=paper_1711_10413_b200/_build/libompds_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab1/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab1/gpu_tests.log
for rep in 1 2; do for v in A B; do lib=$A; [ $v = B ] && lib=$B
 OMPDS_LIB_PATH=$lib PER_SM=16,20,22,24,28,32 timeout 300 python tools/cfg1_sweep.py gpurun_out/ab1/cfg1_${v}_${rep}.json > /dev/null 2>&1
done; done
timeout 900 bash tools/ab_bench.sh $A $B > gpurun_out/ab1/ab_bench.txt 2>&1
