# per-pass ncu launch lists for multi-pass sizes: bash tools/gpu_pass_times.sh prec:logn ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in $@; do
  p=${spec%%:*}; l=${spec##*:}
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/pt_${p}_$l.csv \
    python tools/profile_single.py --prec $p --logn $l --reps 1 > /dev/null 2>&1
done
python tools/pass_times.py gpurun_out/pt_*.csv > gpurun_out/pass_times.txt
