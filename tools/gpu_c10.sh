cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft.py tests/test_gpu_abft.py tests/test_gpu_fix.py tests/test_gpu_campaign.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo rc=$? >> gpurun_out/pytest_sel.log
timeout 1500 python tools/tune.py --sizes 3-13 --prec fp32 --out gpurun_out/tune_r02c_fp32.json > gpurun_out/tune32.log 2>&1
timeout 900 python tools/tune.py --sizes 11-13 --prec fp64 --out gpurun_out/tune_r02c_fp64.json > gpurun_out/tune64.log 2>&1
timeout 900 python bench.py --skip-c3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
