mkdir -p gpurun_out
timeout 300 python scripts/phase_prof.py > gpurun_out/phase_prof.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or concurrent or config1 or cfg1 or overlap" > gpurun_out/fused_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/fused_tests.log
timeout 600 python bench.py --no-secondary --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err
head -n 12 gpurun_out/phase_prof.log; tail -n 3 gpurun_out/fused_tests.log; cut -c1-330 gpurun_out/bench1.json
