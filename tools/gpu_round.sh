set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1000 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncul $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_fused -s 50 -c 1 -o gpurun_out/full -f python tools/profile_step.py --workload c2 --nt 30 --K 2 > gpurun_out/ncu_full.log 2>&1; echo ncuf $?
