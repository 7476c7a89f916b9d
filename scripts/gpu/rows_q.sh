mkdir -p gpurun_out
timeout 300 python scripts/time_stream.py 266 256 32 20 > gpurun_out/time266.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "stream or rows or config0 or cfg0 or config3 or config2" > gpurun_out/rows_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/rows_tests.log
cat gpurun_out/time266.log; tail -n 3 gpurun_out/rows_tests.log
