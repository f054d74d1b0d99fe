#!/bin/bash
# dev-build experiment: N-tile width of the tap-reuse kernel on the C3 layers (batch 64, w1a2)
export APNN_LIB=$PWD/paper_2106_12169_b200/libapnn_s2.so
for L in "56 64 64 1" "56 64 128 2" "28 128 128 1" "28 128 256 2" "14 256 256 1" "14 256 512 2" "7 512 512 1"; do
  set -- $L
  for bn in 64 128 256; do
    echo "H=$1 C=$2 Co=$3 s=$4 bn=$bn: $(APNN_HALO_BN=$bn python scripts/conv_one.py 64 $1 $2 $3 3 $4 1 2 1 2 0 0 10)"
  done
done
