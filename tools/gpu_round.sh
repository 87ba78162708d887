# end-of-round evidence: smoke, the bench line (with the cpu leg), the ncu launch list of the bench command,
# one full capture of the step kernel (tools/profile_summary.py turns them into profiles/<tag>_*)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo benchref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1000 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncul $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_fused -s 50 -c 1 -o gpurun_out/full -f python tools/profile_step.py --workload c2 --nt 30 --K 2 > gpurun_out/ncu_full.log 2>&1; echo ncuf $?
