#!/bin/bash
# times FFMA CTA-tile variants (dconv_cuda_set_ffma_variant) on VGG-like layers
for v in "$@"; do
  echo "variant $v"
  for shp in "64 64 226 226 3 1 32" "256 256 58 58 3 1 32" "128 128 114 114 3 1 32" "512 512 30 30 3 1 32" "512 512 16 16 3 1 32"; do
    python -c "
import sys; sys.path.insert(0, '.')
from paper_1809_10170_b200 import _abi
_abi.lib().dconv_cuda_set_ffma_variant($v)
sys.argv = ['one_layer.py'] + '$shp 2'.split()
exec(open('tools/one_layer.py').read())
" 2>&1 | tail -1
  done
done
