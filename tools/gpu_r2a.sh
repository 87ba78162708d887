timeout 600 python -m pytest tests -m gpu -x -q -k "chunked or block_split or c2_columns" 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python - <<'P'
import json; d=json.load(open('gpurun_out/bench.json'))
print('VALUE', d['value']/1e9, 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value']/1e9, 'med', d['ms_per_step_median'], d['ms_per_step_all'])
print('phases', d['e2e']['phases_ms'], 'mono', d['monodomain'])
P
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --workload c4w1 --steps 2 --warmup 1 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo dist $?
tail -c 1500 gpurun_out/bench_dist1.json; tail -5 gpurun_out/bench_dist1.err
