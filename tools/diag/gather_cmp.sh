# batch-64 graph p50 and in-graph per-function times: PDL on/off
f() { tag=$1; shift; env "$@" python tools/diag/batch_funcs.py --tag $tag $PX 2>&1 | tail -1; }
for PX in "--precision 64" "--precision 32"; do
f default
f nopdl FEWHA_PDL=0
done
