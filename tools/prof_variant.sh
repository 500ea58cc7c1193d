cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for sc in two_sided_group none; do
  o=gpurun_out/v6_fp32_n5_$sc
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k regex:"fft_single_kernel<float" -c 1 -o $o -f python tools/profile_single.py --prec fp32 --logn 5 --scheme $sc --reps 2 --variant 6 > $o.log 2>&1
  python tools/ncu_summary.py $o.ncu-rep > $o.md 2>&1
  python tools/sass_hot.py $o.ncu-rep --top 25 --lines 30 > $o.sass.txt 2>&1
done
