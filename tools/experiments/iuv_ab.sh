ST_IUV_VARIANT=4 python -m pytest tests -m gpu -q -x -k "engine or rtpm or iuv or large or cpd or c3" 2>&1 | tail -2
for i in 1 2; do for v in 1 4; do echo -n "v$v "; ST_IUV_VARIANT=$v python tools/prof_spectral.py --reps 3 --which c3; done; done
