cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for s in 1 0; do echo "INV_STAGE=$s"; FEWHA_INV_STAGE=$s python scratch/timing.py 2>&1 | sed -n 3,3p; FEWHA_INV_STAGE=$s python tools/profile_frame.py --batch 64 --frames 3 | tail -1; done
python scratch/timing.py 2>&1 | sed -n 3,4p
