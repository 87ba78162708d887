# build experiment variants of libkfp.so in parallel: tools/build_variants.sh name:FLAGS ...
cd /root/repo
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
      -I include --cudart=static $flags -o build/var_$name.so paper_1306_4596_b200/csrc/kfp_api.cu > /tmp/var_$name.log 2>&1 \
      && echo "built $name" || { echo "FAILED $name"; tail -5 /tmp/var_$name.log; } ) &
done
wait
