#!/bin/bash
# Profiles for profiles/: launch list of the bench command + ncu --set full of the top kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/ncu_gemm_fc -f \
    python tools/gemm_one.py 4096x3072x768 0 0 -1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/ncu_gemm_8192 -f \
    python tools/gemm_one.py 8192x8192x8192 0 0 -1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_kernel -s 1 -c 1 -o gpurun_out/ncu_leaf -f \
    python tools/commit_one.py > /dev/null 2>&1
ls -la gpurun_out
