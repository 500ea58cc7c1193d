# ncu --set full of one single-kernel VARIANT (tfft_tune_select), ABFT on vs off:
#   PREC=fp32 LOGN=5 VARIANT=6 bash tools/prof_variant.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
P=${PREC:-fp32}; L=${LOGN:-5}; V=${VARIANT:-0}
for sc in two_sided_group none; do
  o=gpurun_out/v${V}_${P}_n${L}_$sc
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k regex:"fft_single_kernel<" -c 1 -o $o -f \
    python tools/profile_single.py --prec $P --logn $L --scheme $sc --reps 2 --variant $V > $o.log 2>&1
  python tools/ncu_summary.py $o.ncu-rep > $o.md 2>&1
  python tools/sass_hot.py $o.ncu-rep --top 25 --lines 30 > $o.sass.txt 2>&1
done
