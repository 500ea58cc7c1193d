# closed-form e^T W (multi-pass first pass): parity tests, per-pass ncu times
# vs the table build (AB_LIB), and the C3 leg of the bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_etw.py tests/test_gpu_fft.py tests/test_gpu_abft.py tests/test_gpu_campaign.py -x -q > gpurun_out/pytest_cf.log 2>&1; echo rc=$? >> gpurun_out/pytest_cf.log
for spec in fp64:20 fp64:23 fp64:25 fp32:16 fp32:20 fp32:25; do
  IFS=: read p l <<< "$spec"
  for lib in product $AB_LIB; do
    tag=$(basename $lib .so)
    if [ "$lib" = product ]; then unset TFFT_LIB_PATH; else export TFFT_LIB_PATH=$lib; fi
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"fft_pass|finalize" --csv --log-file gpurun_out/cf_${tag}_${p}_$l.csv python tools/profile_single.py --prec $p --logn $l --reps 1 > /dev/null 2>&1
    echo "== $tag $p 2^$l" >> gpurun_out/pass_cf.txt
    python tools/pass_times.py gpurun_out/cf_${tag}_${p}_$l.csv | tail -4 >> gpurun_out/pass_cf.txt 2>&1
  done
done
unset TFFT_LIB_PATH
rm -f gpurun_out/cf_*.csv
timeout 900 python bench.py --skip-cpu > gpurun_out/bench_cf.log 2>&1
