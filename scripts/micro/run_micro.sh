#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/stagein scripts/micro/stagein.cu -lcuda && /tmp/stagein > gpurun_out/m_stagein.txt 2>&1
