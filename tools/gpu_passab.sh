# per-pass times (ncu launch list) of fp64 2^24 / 2^25, product build vs an
# ablation build (AB_LIB): the cost of the first pass's e^T W loads
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for l in 24 25; do
  for lib in product ${AB_LIB:-}; do
    tag=$(basename $lib .so)
    if [ "$lib" = product ]; then unset TFFT_LIB_PATH; else export TFFT_LIB_PATH=$lib; fi
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/pass_${tag}_fp64_$l.csv python tools/profile_single.py --prec fp64 --logn $l --reps 1 > /dev/null 2>&1
    python tools/pass_times.py gpurun_out/pass_${tag}_fp64_$l.csv >> gpurun_out/pass_ab.txt 2>&1
  done
done
unset TFFT_LIB_PATH
