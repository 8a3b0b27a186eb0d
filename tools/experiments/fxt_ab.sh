#!/bin/bash
# usage: bash tools/experiments/fxt_ab.sh  (on the GPU box)
cd "$(dirname "$0")/../.."
Q=tools/experiments/quads_c4.bin
for i in 1 2; do
python tools/experiments/fxt_ab.py 4 30
ST_FXT=2 python tools/experiments/fxt_ab.py 4 30
ST_FXT=2 ST_FXT_QUADS=$Q python tools/experiments/fxt_ab.py 4 30
ST_FXT=3 ST_FXT_QUADS=$Q python tools/experiments/fxt_ab.py 4 30
ST_FXT=1 ST_FXT_QUADS=$Q python tools/experiments/fxt_ab.py 4 30
done
ST_FXT=2 ST_FXT_QUADS=$Q python tools/experiments/fxt_ab.py 1 30
python tools/experiments/fxt_ab.py 1 30
