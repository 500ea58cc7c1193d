# correctness of the changed kernels, then the single-kernel tuner on the sizes
# of a TFFT_TUNE_SIZES tuning build (logs + json only: small gpurun_out);
# AB_LIB=path also times an experiment build on AB_SIZES.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft.py tests/test_gpu_abft.py tests/test_gpu_fix.py tests/test_gpu_campaign.py -x -q > gpurun_out/pytest_tune.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tune.log
timeout 1500 python tools/tune.py --sizes ${TUNE32:-5-13} --prec fp32 --out gpurun_out/tune_r02_fp32.json > gpurun_out/tune32.log 2>&1
if [ -n "$TUNE64" ]; then
timeout 900 python tools/tune.py --sizes ${TUNE64} --prec fp64 --out gpurun_out/tune_r02_fp64.json > gpurun_out/tune64.log 2>&1
fi
if [ -n "$AB_LIB" ]; then
TFFT_LIB_PATH=$AB_LIB timeout 900 python tools/tune.py --sizes ${AB_SIZES:-5-10} --prec fp32 --out gpurun_out/tune_r02_ab.json > gpurun_out/tune_ab.log 2>&1
fi
du -sh gpurun_out; ls gpurun_out
