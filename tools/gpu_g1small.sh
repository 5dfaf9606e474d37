#!/bin/bash
# G1 tile plans at the c4 rank shapes (M = 1170 / 585): forced BN / mode vs the planner.
export PYTHONPATH=$PWD
for W in 4 8; do
  echo "== W=$W planner"; python tools/gemm_probe.py c4 --ranks $W 2>&1 | grep '^{'
  for m in 1 3; do for bn in 128 192 256; do
    [ $m = 3 ] && [ $bn = 192 ] && continue
    echo "== W=$W mode=$m bn=$bn"; IFX_G1_MODE=$m IFX_G1_BN=$bn python tools/gemm_probe.py c4 --ranks $W 2>&1 | grep '^{'
  done; done
done
