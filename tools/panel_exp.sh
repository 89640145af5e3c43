#!/bin/bash
# Panel column-loop timing experiments (single CTA, clock64): product code vs dev variants.
cd tools
for V in "" "-DTQR_PF_SKIP_NONCRIT"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 $V panel_bench.cu -o /tmp/pb 2>/dev/null && echo "== variant '$V'" && /tmp/pb | grep panel_factor | grep -v OLD
done
