# k_plane iteration: phase stamps, config-2 parity tests, config-2 bench line
mkdir -p gpurun_out
timeout 300 python scripts/plane_prof.py > gpurun_out/plane_prof.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "plane or config2 or stream or cfg2 or config_2" > gpurun_out/plane_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/plane_tests.log
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
cat gpurun_out/plane_prof.log; tail -n 3 gpurun_out/plane_tests.log; cut -c1-300 gpurun_out/bench_cfg2.json
