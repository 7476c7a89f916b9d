# ncu --set full of the config-4 kernels at one K (accumulate, Cholesky, row solve); K from $1
K=${1:-256}
mkdir -p gpurun_out
timeout 300 python bench.py --config 4 --ks $K --steps 3 --warmup 1 > gpurun_out/cfg4_$K.json 2>&1; cut -c1-400 gpurun_out/cfg4_$K.json
for k in k_chol_blocked k_hist_accum_tc k_rowsolve_chol; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/cfg4_${K}_$k -f python bench.py --config 4 --ks $K --steps 1 --warmup 0 > gpurun_out/ncu_cfg4_${K}_$k.log 2>&1
  echo "$k rc=$?"
done
