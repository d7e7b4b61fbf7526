#!/bin/bash
# One GPU call: build, parity tests, bench, ncu launch list, ncu full capture of the top kernel.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q ${TESTS:-} > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1; wc -l gpurun_out/launches.csv
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-gemm_kernel} -s ${KSKIP:-15} -c 1 \
      -o gpurun_out/prof_top -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
fi
