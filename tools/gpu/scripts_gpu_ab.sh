#!/bin/bash
# A/B of an alternative in-tree build (OZ2_LIB): GPU tests on it, then kscan / midsize / bench for both
ALT=${ALT:-paper_2504_08009_b200/liboz2_u2.so}
OZ2_LIB=$(realpath $ALT) timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for i in 1 2; do
for lib in paper_2504_08009_b200/liboz2.so $ALT; do
  echo "== $lib"
  OZ2_LIB=$(realpath $lib) timeout 300 python tools/kscan.py
  OZ2_LIB=$(realpath $lib) timeout 300 python tools/midsize.py 4096,8192
done; done
