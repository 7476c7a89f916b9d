# blocked Cholesky at config-4 shapes vs CTAs per SM (OCSC_CHOL_MINSMEM) and CTA width (OCSC_CHOL_NT)
mkdir -p gpurun_out
run() {
  env $1 timeout 300 python bench.py --config 4 --ks $2 --steps 3 --warmup 1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', d['K'], {k: round(v,2) for k,v in d['ms'].items()}, 'err %.1e' % d['parity_rel_err_vs_dense_c128'])
"
}
run OCSC_CHOL_MINSMEM=0 256
run OCSC_CHOL_MINSMEM=100000 256
run OCSC_CHOL_MINSMEM=200000 256
run "OCSC_CHOL_NT=256 OCSC_CHOL_MINSMEM=100000" 256
run "OCSC_CHOL_NT=512 OCSC_CHOL_MINSMEM=200000" 256
run OCSC_CHOL_MINSMEM=0 512
run "OCSC_CHOL_NT=256 OCSC_CHOL_MINSMEM=0" 512
