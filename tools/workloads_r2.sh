# one bench line per workload (kernel rate, roofline, e2e) on the round's code -> gpurun_out/wl_<name>.json
for w in c0 c1 c2 c3 c4w1 paper_j4; do
  timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu --workload $w > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err
  echo "$w rc $?"
done
