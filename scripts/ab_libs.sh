#!/bin/bash
# same-box A/B of two builds of libapnn (APNN_LIB) on conv layers: ./scripts/ab_libs.sh libA libB
for L in "$1" "$2"; do
  export APNN_LIB=$PWD/paper_2106_12169_b200/$L
  echo "$L: vgg_c4 $(python scripts/conv_one.py 256 56 256 256 3 1 1 2 1 2 2 2 5) vgg_c7 $(python scripts/conv_one.py 256 28 384 384 3 1 1 2 1 2 2 2 5) R18L1 $(python scripts/conv_one.py 1024 56 64 64 3 1 1 8 2 0 8 0 3) R18L3 $(python scripts/conv_one.py 1024 14 256 256 3 1 1 8 2 0 8 0 3) C3L1 $(python scripts/conv_one.py 64 56 64 64 3 1 1 2 1 2 0 0 10) C3L3 $(python scripts/conv_one.py 64 14 256 256 3 1 1 2 1 2 0 0 10)"
done
