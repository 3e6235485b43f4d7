# batch-64 graph p50 and in-graph per-function times under several gather settings
f() { tag=$1; shift; env "$@" python tools/diag/batch_funcs.py --tag $tag $PX 2>&1 | tail -1; }
export FEWHA_GATHER_LATE=1
for PX in "--precision 64" "--precision 32"; do
f d4m2 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=2
f d4m3 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=3
f d4m4 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=4
f d2m3 FEWHA_GATHER_NI=2 FEWHA_GATHER_MINB=3
f d2m4 FEWHA_GATHER_NI=2 FEWHA_GATHER_MINB=4
f d4m2r4 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=2 FEWHA_GATHER_ROWS=4
f d4m4r4 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=4 FEWHA_GATHER_ROWS=4
done
unset FEWHA_GATHER_LATE
for d in 0 1; do for m in 2 3; do echo "single direct $d minb $m"; FEWHA_GATHER_DIRECT=$d FEWHA_GATHER_MINB=$m python tools/diag/ab_lat.py --frames 600 | tail -1; done; done
FEWHA_GATHER_DIRECT=1 FEWHA_GATHER_ROWS=8 python tools/diag/ab_lat.py --frames 600 | tail -1
