#!/bin/bash
# Experiment builds: rebuild the single-kernel parts holding N = 2048 (part 3),
# 4096 (part 0) and 8192 (part 1) with extra -D flags and link
# paper_2405_02520_b200/ablate/libtfft_<tag>.so from the product objects.
#   bash tools/ablate_build.sh TAG "-DTFFT_ABLATE=1" [TAG2 "-D..."] ...
# PARTS="0 1 2 3" rebuilds other fp32 parts (default 0 1 3).
set -e
cd "$(dirname "$0")/../paper_2405_02520_b200"
mkdir -p ablate build/ablate
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I../include -Icsrc"
args=("$@")
for ((i = 0; i < ${#args[@]}; i += 2)); do
  tag=${args[i]}; flags=${args[i+1]}
  for p in ${PARTS:-0 1 3}; do
    $NV $flags -c csrc/gen_single_fp32_$p.cu -o build/ablate/gen_single_fp32_${p}_$tag.o &
  done
done
wait
for ((i = 0; i < ${#args[@]}; i += 2)); do
  tag=${args[i]}
  pat=$(echo ${PARTS:-0 1 3} | tr -d ' ')
  objs=$(ls build/*.o | grep -v "gen_single_fp32_[$pat].o")
  mine=$(for p in ${PARTS:-0 1 3}; do echo build/ablate/gen_single_fp32_${p}_$tag.o; done)
  $NV -shared -o ablate/libtfft_$tag.so $objs $mine -lcudart
done
ls -la ablate
