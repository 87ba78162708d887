# bench every gpurun_out/var_*.so on c2 (short runs); prints value / frac per variant
for so in build/var_*.so; do
  n=$(basename $so .so)
  KFP_LIB_PATH=$so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$n.json 2>gpurun_out/b_$n.err
  python -c "import json,sys; d=json.load(open('gpurun_out/b_$n.json')); print('$n', round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline']['avg_launch_us'])" || echo "$n failed"
done
