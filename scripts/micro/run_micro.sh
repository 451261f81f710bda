#!/bin/bash
mkdir -p gpurun_out
[ -n "$SKIP_STAGEIN" ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/stagein scripts/micro/stagein.cu -lcuda && /tmp/stagein > gpurun_out/m_stagein.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/empty scripts/micro/empty.cu && /tmp/empty > gpurun_out/m_empty.txt 2>&1
