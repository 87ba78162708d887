# GPU suite + smoke, then the default bench line (N=1) and the reference arm
bash tools/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value']/1e9, d['roofline']['frac'], d['e2e']['value']/1e9, d['e2e']['value']/d['value'], d['e2e']['phases_ms'])"
