#!/bin/bash
# Builds librd variants that differ only in one GEMM unit's compile flags (default the TMA
# PM-stats unit; AB_UNIT=rd_gemm_pm_stats for the cp.async one), for same-session A/B timing
# (RD_LIB=paper_2409_17658_b200/librd_<tag>.so).
#   [AB_UNIT=<unit>] tools/build_ab.sh <tag> <extra nvcc flags...>
set -eu
TAG=$1; shift
B=paper_2409_17658_b200/build
U=${AB_UNIT:-rd_gemm_pm_stats_tma}
python -m paper_2409_17658_b200.build > /dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp \
  -I include "$@" -c paper_2409_17658_b200/csrc/$U.cu -o /tmp/ab_$TAG.o
objs=$(ls $B/*.o | grep -v "/$U.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs /tmp/ab_$TAG.o \
  -o paper_2409_17658_b200/librd_$TAG.so -lgomp -lpthread
echo paper_2409_17658_b200/librd_$TAG.so
