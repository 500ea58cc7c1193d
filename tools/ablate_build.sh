#!/bin/bash
# Cost attribution of the fused ABFT: rebuild the single-kernel parts holding
# N=2048 (part 3) and N=4096 (part 0) with -DTFFT_ABLATE=k and link
# paper_2405_02520_b200/ablate/libtfft_k.so from the product objects.
set -e
cd "$(dirname "$0")/../paper_2405_02520_b200"
mkdir -p ablate build/ablate
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I../include -Icsrc"
for k in "$@"; do
  for p in 0 3; do
    $NV -DTFFT_ABLATE=$k -c csrc/gen_single_fp32_$p.cu -o build/ablate/gen_single_fp32_${p}_$k.o &
  done
done
wait
for k in "$@"; do
  objs=$(ls build/*.o | grep -v "gen_single_fp32_0.o\|gen_single_fp32_3.o")
  $NV -shared -o ablate/libtfft_$k.so $objs build/ablate/gen_single_fp32_0_$k.o build/ablate/gen_single_fp32_3_$k.o -lcudart
done
ls -la ablate
