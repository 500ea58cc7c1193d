# The round-end driver sequence plus evidence: pytest -m gpu, smoke, bench,
# the bench launch list under ncu, and ncu --set full summaries (reports are
# deleted on the box; only .md/.sass.txt summaries come back).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --skip-cpu > gpurun_out/bench_ncu.log 2>&1
fi
if [ -n "$PROF32" ]; then COUNT=2 bash tools/gpu_prof.sh ${PTAG:-r02} $PROF32 > gpurun_out/prof32.log 2>&1; fi
if [ -n "$PROF64" ]; then COUNT=5 bash tools/gpu_prof.sh ${PTAG:-r02} $PROF64 > gpurun_out/prof64.log 2>&1; fi
du -sh gpurun_out; ls gpurun_out
