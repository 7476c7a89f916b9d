# fused-kernel iteration loop: parity tests of the fused paths, phase stamps, headline bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or cfg1 or headline or smoke" > gpurun_out/gt_fused.txt 2>&1; tail -3 gpurun_out/gt_fused.txt
timeout 300 python scripts/phase_prof.py > gpurun_out/phase.txt 2>&1; head -12 gpurun_out/phase.txt
timeout 300 python bench.py --no-secondary > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; cut -c1-400 gpurun_out/bench_c.json; tail -3 gpurun_out/bench_c.err
