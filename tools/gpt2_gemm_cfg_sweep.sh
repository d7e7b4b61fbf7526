#!/bin/bash
# per-shape R-GEMM time of the GPT-2 step under every forced tile configuration
# (tools/gpt2_gemm_shapes.py with FORCE_CFG), plus the automatic choice
mkdir -p gpurun_out
{ echo "cfg auto"; timeout 200 python tools/gpt2_gemm_shapes.py; } > gpurun_out/cfg_sweep.txt 2>&1
for c in $(seq 0 18); do
  { echo "cfg $c"; FORCE_CFG=$c timeout 200 python tools/gpt2_gemm_shapes.py; } >> gpurun_out/cfg_sweep.txt 2>&1
done
