#!/bin/bash
# A/B the kernel variants built under .variants/<name>/librfg.so (see
# tools/stage_bench.py); run on the GPU box from the repo root.
for d in .variants/*/; do
  RFG_LIB_PATH=$PWD/${d}librfg.so python tools/stage_bench.py 2>&1 | tail -1
done
