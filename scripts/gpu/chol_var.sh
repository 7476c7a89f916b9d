# Cholesky variants: parity tests, then config 4 at K = 256 / 512 per CTA width (OCSC_CHOL_NT)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "chol or Chol or history or rowsolve" > gpurun_out/gt_chol.txt 2>&1; tail -2 gpurun_out/gt_chol.txt
for nt in 128 256 512; do
  OCSC_CHOL_NT=$nt timeout 300 python bench.py --config 4 --ks 256 512 --steps 3 --warmup 1 > gpurun_out/cfg4_nt$nt.json 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/cfg4_nt$nt.json'):
    if l.startswith('{'):
        d=json.loads(l); print('NT=$nt', d['K'], {k: round(v,2) for k,v in d['ms'].items()}, 'err', d['parity_rel_err_vs_dense_c128'])
"
done
