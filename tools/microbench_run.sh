#!/bin/bash
# Build and run the diagnostic microbenchmarks (launch floor, L2 bandwidth) on the GPU box.
set -e
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/floor tools/microbench_floor.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/l2bw tools/microbench_l2.cu
/tmp/floor | tee gpurun_out/microbench_floor.txt
/tmp/l2bw | tee gpurun_out/microbench_l2.txt
