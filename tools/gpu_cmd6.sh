cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or c2_full or c3_full or deterministic or block_split or translation" > gpurun_out/t_prod.log 2>&1; echo "prod tests rc=$? $(tail -1 gpurun_out/t_prod.log)"
WLS="c2 c4w1 c3" bash tools/var_round.sh 2>&1 | grep -v "tests rc"
