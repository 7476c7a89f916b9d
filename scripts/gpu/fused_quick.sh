# fused-kernel timing only: phase stamps and the headline bench
mkdir -p gpurun_out
timeout 300 python scripts/phase_prof.py > gpurun_out/phase.txt 2>&1; head -12 gpurun_out/phase.txt
timeout 300 python bench.py --no-secondary > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; cut -c1-300 gpurun_out/bench_c.json; tail -3 gpurun_out/bench_c.err
