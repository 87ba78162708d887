# experiment round: parity subset + c2/c3/c4w1 bench of the product library and every build/var_*.so
cd /root/repo
mkdir -p gpurun_out
for so in $(ls build/var_*.so 2>/dev/null | grep -v abl_); do
  n=$(basename $so .so)
  KFP_LIB_PATH=$so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or c2_full or c3_full or deterministic" > gpurun_out/t_$n.log 2>&1; echo "$n tests rc=$? $(tail -1 gpurun_out/t_$n.log)"
done
for wl in ${WLS:-c2 c3 c4w1}; do
  for so in paper_1306_4596_b200/libkfp.so build/*var_*.so; do
    n=$(basename $so .so)
    KFP_LIB_PATH=$so timeout 300 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_${n}_$wl.json 2>gpurun_out/b_${n}_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/b_${n}_$wl.json')); print('$wl $n', round(d['value']/1e9,1), round(d['roofline']['frac'],3), round(d['roofline']['avg_launch_us'],2), d['config']['plan'])" || { echo "$wl $n failed"; tail -3 gpurun_out/b_${n}_$wl.err; }
  done
done
