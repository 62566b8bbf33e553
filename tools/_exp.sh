timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu4.log 2>&1
for n in 1 2 4; do timeout 300 python tools/cluster_bench.py $n weak 30 > gpurun_out/cl_w$n.log 2>&1; done
for n in 2 4; do timeout 300 python tools/cluster_bench.py $n strong 30 > gpurun_out/cl_s$n.log 2>&1; done
