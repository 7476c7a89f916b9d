# config-4 bench lines at every K and ncu captures of the history kernels (K = 256, 512)
mkdir -p gpurun_out
timeout 300 python bench.py --config 4 --steps 5 --warmup 2 > gpurun_out/cfg4_all.jsonl 2> gpurun_out/cfg4_all.err
for K in 256 512; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chol_blocked|k_hist_accum_tc" -c 2 \
    -o gpurun_out/hist_$K -f python scripts/chol_prof.py $K > gpurun_out/ncu_hist_$K.log 2>&1
  echo "K=$K rc=$?"
done
