#!/bin/bash
# A/B timing of alternative library builds (tools/lib_*.so) on representative layers
for L in tools/lib_*.so; do
  echo "== $L"
  for shp in "64 64 226 226 3 1 32" "256 256 58 58 3 1 32" "128 128 114 114 3 1 32" "512 512 30 30 3 1 32" "512 512 16 16 3 1 32" "256 64 56 56 1 1 32"; do
    DCONV_LIB=$L python tools/one_layer.py $shp 2
  done
done
