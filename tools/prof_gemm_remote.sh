#!/bin/bash
# ncu --set full of R-GEMM configurations; summaries written remotely (reports are large)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
mkdir -p gpurun_out/prof_tmp
for spec in "$@"; do
  set -- $spec
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -s 2 -c 1 \
      -o gpurun_out/prof_tmp/$5 -f python tools/gemm_one.py $1 $2 $3 $4 > /dev/null 2>&1
  ncu -i gpurun_out/prof_tmp/$5.ncu-rep --page raw --csv > gpurun_out/prof_tmp/$5.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/prof_tmp/$5.csv > gpurun_out/ncu_$5.txt
  ncu -i gpurun_out/prof_tmp/$5.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tmp/$5_src.csv 2>/dev/null
  python tools/sass_stalls.py gpurun_out/prof_tmp/$5_src.csv >> gpurun_out/ncu_$5.txt
done
rm -rf gpurun_out/prof_tmp
