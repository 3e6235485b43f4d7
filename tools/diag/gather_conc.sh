# fp64 batch: gather instances per CTA / residency with 1 and 2 engines (two streams)
set -u
for cfg in "4 2" "2 3" "1 4" "2 2"; do
  set -- $cfg
  echo "gather NI $1 MINB $2:"
  FEWHA_GATHER_NI=$1 FEWHA_GATHER_MINB=$2 timeout 300 python tools/batch_sweep.py --sizes 32,64 --precision 64 2>&1 | grep concurrent
done
