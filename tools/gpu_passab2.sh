# first-pass tile order A/B (TFFT_POS_CHUNKS=0 vs default) on fp64 2^20..2^25 + fp32 2^20/2^25:
# ncu per-pass times, then the GPU parity tests of the multi-pass path
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in fp64:20 fp64:23 fp64:24 fp64:25 fp32:20 fp32:25; do
  IFS=: read p l <<< "$spec"
  for pc in 0 1; do
    TFFT_POS_CHUNKS=$pc timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"fft_pass|finalize" --csv --log-file gpurun_out/pc${pc}_${p}_$l.csv python tools/profile_single.py --prec $p --logn $l --reps 1 > /dev/null 2>&1
    echo "== pos_chunks=$pc $p 2^$l" >> gpurun_out/pass_ab2.txt
    python tools/pass_times.py gpurun_out/pc${pc}_${p}_$l.csv >> gpurun_out/pass_ab2.txt 2>&1
  done
done
rm -f gpurun_out/pc*.csv
timeout 900 python -m pytest tests/test_gpu_fft.py tests/test_gpu_abft.py tests/test_gpu_campaign.py tests/test_gpu_scale.py -x -q -k "multi or pass or campaign or c3 or fp64 or large or 2_" > gpurun_out/pytest_pass.log 2>&1; echo rc=$? >> gpurun_out/pytest_pass.log
