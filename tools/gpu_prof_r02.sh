# round-2 evidence run: selected parity tests, the bench launch list, ncu
# summaries of the dominant single kernels (fp32) and the fp64 single/C3
# kernels (pipe utilisation); TUNE=1 adds the single-kernel tuner on the
# sizes of a TFFT_TUNE_SIZES build.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests/test_gpu_fix.py tests/test_gpu_scale.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
fi
if [ -z "$NO_PROF" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --skip-cpu --skip-c3 > gpurun_out/bench_ncu.log 2>&1
COUNT=2 bash tools/gpu_prof.sh r02 ${PROF32:-fp32:5 fp32:6 fp32:11 fp32:12 fp32:13} > gpurun_out/prof32.log 2>&1
COUNT=5 bash tools/gpu_prof.sh r02 ${PROF64:-fp64:13 fp64:20 fp64:25} > gpurun_out/prof64.log 2>&1
fi
if [ -n "$TUNE" ]; then
  timeout 1200 python tools/tune.py --sizes ${TUNE32:-11-13} --prec fp32 --out gpurun_out/tune_r02_fp32.json > gpurun_out/tune32.log 2>&1
  timeout 900 python tools/tune.py --sizes ${TUNE64:-11-12} --prec fp64 --out gpurun_out/tune_r02_fp64.json > gpurun_out/tune64.log 2>&1
fi
du -sh gpurun_out; ls gpurun_out
