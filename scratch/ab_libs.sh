for g in 9 7 5; do cp scratch/libs/lib_g$g.so paper_2009_00946_b200/lib/libfewha_gpu.so; echo "G=$g"; python tools/diag/ab.py "{}"; done
