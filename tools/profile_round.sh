#!/bin/bash
# One gpurun call producing the judged profiles (summaries are written remotely: .ncu-rep files are large).
#  gpurun_out/launches.csv : ncu launch list of the bench command (duration + DRAM bytes per launch)
#  gpurun_out/ncu_<tag>.txt: ncu --set full summaries (+ per-SASS stall attribution) of the top kernels
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/launches_bench.log 2>&1
echo "launch list: $(wc -l < gpurun_out/launches.csv) lines"
python tools/launch_shares.py gpurun_out/launches.csv 0 embedding_kernel 3 > gpurun_out/launch_shares.txt 2>&1
bash tools/prof_gemm_remote.sh "4096x768x3072 1 0 -1 gemm_fc2_tn" "4096x3072x768 1 0 -1 gemm_fc_tn" \
    "8192x8192x8192 1 0 -1 gemm_8192_tn" "8192x8192x8192 0 0 -1 gemm_8192_nn" "4096x50304x768 1 0 -1 gemm_lmhead_tn" \
    "512x512x64 0 1 -1 gemm_scores_nt"
bash tools/prof_cublas_remote.sh 8192x8192x8192 1 0 cublas_8192_tn
mkdir -p gpurun_out/prof_tmp
for k in 0 1 2; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -s $((3 + k)) -c 1 \
      -o gpurun_out/prof_tmp/attn$k -f python tools/attn_one.py > /dev/null 2>&1
  ncu -i gpurun_out/prof_tmp/attn$k.ncu-rep --page raw --csv > gpurun_out/prof_tmp/attn$k.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/prof_tmp/attn$k.csv > gpurun_out/ncu_gemm_attn$k.txt
done
mkdir -p gpurun_out/prof_tmp
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_probs -s 2 -c 1 \
    -o gpurun_out/prof_tmp/probs -f python tools/attn_probs_one.py > /dev/null 2>&1
ncu -i gpurun_out/prof_tmp/probs.ncu-rep --page raw --csv > gpurun_out/prof_tmp/probs.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_tmp/probs.csv > gpurun_out/ncu_attn_probs.txt
ncu -i gpurun_out/prof_tmp/probs.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tmp/probs_src.csv 2>/dev/null
python tools/sass_stalls.py gpurun_out/prof_tmp/probs_src.csv >> gpurun_out/ncu_attn_probs.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:leaf_kernel -s 1 -c 1 \
    -o gpurun_out/prof_tmp/leaf -f python tools/commit_one.py > /dev/null 2>&1
ncu -i gpurun_out/prof_tmp/leaf.ncu-rep --page raw --csv > gpurun_out/prof_tmp/leaf.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_tmp/leaf.csv > gpurun_out/ncu_leaf.txt
rm -rf gpurun_out/prof_tmp
ls -la gpurun_out/ncu_*.txt
