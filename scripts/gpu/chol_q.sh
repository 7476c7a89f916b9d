mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "chol or Chol or history or rowsolve or config3 or cfg3 or K120 or any_k" > gpurun_out/gt_chol.txt 2>&1; echo "pytest exit $?" >> gpurun_out/gt_chol.txt
timeout 300 python scripts/chol_prof.py 256 512 > gpurun_out/chol_prof.log 2>&1
timeout 300 python bench.py --config 4 --steps 5 --warmup 2 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err
tail -n 3 gpurun_out/gt_chol.txt; cat gpurun_out/chol_prof.log; python - <<'PY'
import json
for l in open('gpurun_out/cfg4.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['K'], {k: round(v,2) for k,v in d['ms'].items()}, 'err', d['parity_rel_err_vs_dense_c128'], 'fp32', round(d['cholesky_solve']['frac_fp32'],3))
PY
