# End-of-round evidence: the driver sequence (pytest -m gpu, smoke, bench) plus
# the bench launch list with DRAM bytes (-> profiles/traffic_r02.json, read by
# bench.py for roofline.traffic) and ncu --set full summaries of the kernels
# the bench's headline rests on.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_dram.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-c3 > gpurun_out/bench_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches_dram.csv gpurun_out/launches_r02.md gpurun_out/traffic_r02.json > gpurun_out/launch_summary.log 2>&1
cp gpurun_out/traffic_r02.json profiles/traffic_r02.json 2>/dev/null
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
COUNT=2 bash tools/gpu_prof.sh r02c ${PROF32:-fp32:5 fp32:11 fp32:12 fp32:13} > gpurun_out/prof32.log 2>&1
COUNT=5 bash tools/gpu_prof.sh r02c ${PROF64:-fp64:25} > gpurun_out/prof64.log 2>&1
du -sh gpurun_out
