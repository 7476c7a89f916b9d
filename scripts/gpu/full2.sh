# full GPU check: smoke, pytest -m gpu, headline bench (with secondary configs), reference arm,
# launch list of the headline bench, config 4 at every K
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
tail -n 3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-400 gpurun_out/bench.json; tail -n 3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-300 gpurun_out/bench_ref.json
timeout 600 python bench.py --config 4 --steps 5 --warmup 2 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err
timeout 600 python bench.py --config 3 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; cut -c1-300 gpurun_out/cfg3.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo done
