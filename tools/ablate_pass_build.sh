#!/bin/bash
# Experiment builds of the multi-pass kernels: bash tools/ablate_pass_build.sh TAG "-D..." ...
set -e
cd "$(dirname "$0")/../paper_2405_02520_b200"
mkdir -p ablate build/ablate
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I../include -Icsrc"
args=("$@")
for ((i = 0; i < ${#args[@]}; i += 2)); do
  tag=${args[i]}; flags=${args[i+1]}
  for p in fp32 fp64; do $NV $flags -c csrc/gen_pass_$p.cu -o build/ablate/gen_pass_${p}_$tag.o & done
done
wait
for ((i = 0; i < ${#args[@]}; i += 2)); do
  tag=${args[i]}
  objs=$(ls build/*.o | grep -v "gen_pass_fp")
  $NV -shared -o ablate/libtfft_$tag.so $objs build/ablate/gen_pass_fp32_$tag.o build/ablate/gen_pass_fp64_$tag.o -lcudart
done
