# ncu --set full of the multi-pass kernels (first reps), ABFT on vs off: bash tools/gpu_prof_multi.sh TAG prec:logn ...
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=$1; shift
for spec in $@; do
  p=${spec%%:*}; l=${spec##*:}
  for sc in two_sided_group none; do
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"fft_pass_kernel|abft_finalize" -c 8 \
      -o gpurun_out/${TAG}_${p}_n${l}_${sc} -f python tools/profile_single.py --prec $p --logn $l --scheme $sc --reps 2 > gpurun_out/${TAG}_${p}_n${l}_${sc}.log 2>&1
  done
done
