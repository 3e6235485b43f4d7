# per-function mean launch time (ncu launch list, 1 batch-64 frame) under several gather settings
P64="python tools/profile_frame.py --batch 64 --frames 1"
M="--metrics gpu__time_duration.sum --clock-control none --csv"
run() { tag=$1; shift; env "$@" ncu $M -s 42 -c 21 --log-file gpurun_out/lc_$tag.csv $P64 > /dev/null 2>&1; }
run old FEWHA_GATHER_DIRECT=0
run d2m3 FEWHA_GATHER_NI=2 FEWHA_GATHER_MINB=3
run d4m2 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=2
run d4m4 FEWHA_GATHER_NI=4 FEWHA_GATHER_MINB=4
