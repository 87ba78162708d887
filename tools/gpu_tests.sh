# GPU test suite + smoke (optionally a -k filter as $1)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
if [ -n "$1" ]; then K="-k $1"; else K=""; fi
timeout 1500 python -m pytest tests -m gpu -x -q $K --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -25 gpurun_out/pytest_gpu.log
