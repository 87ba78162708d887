"""Cluster-size sweep (KFP_FORCE_C) on one workload (debugging aid): python tools/dbg/cl_sweep.py c4w1 4 8"""
import sys, os, subprocess, json
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
wl = sys.argv[1]
for c in sys.argv[2:]:
    env = dict(os.environ, KFP_FORCE_C=c)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", wl, "--steps", "2", "--warmup", "2",
                          "--no-cpu"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(f"{wl} C={c}: {d['value']/1e9:7.1f} G upd/s frac {d['roofline']['frac']:.3f} {d['config']['plan']}", flush=True)
    except Exception:
        print(wl, c, out.stderr[-500:], flush=True)
