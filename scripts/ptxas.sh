#!/bin/bash
# usage: ./scripts_ptxas.sh file.cu [grep-pattern] — register/spill report for sm_100a
SP=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -c paper_2412_20379_b200/csrc/$1 -I include -I paper_2412_20379_b200/csrc -I $SP/nccl/include -I $SP/cublas/include -o /tmp/ptxas_check.o 2>&1 | grep -E "error|Compiling|registers|spill" | paste - - - | sed 's/ptxas info    ://g' | grep -E "${2:-.}|error" | sed 's/.*Compiling entry function//' | cut -c1-200
