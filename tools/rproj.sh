# ResNet-50 projection shortcuts (1x1, stride 1 and 2) at batch 256, both CTA tiles
cd /root/repo
for shp in "64 256 56 56 1 1 256" "256 512 55 55 1 2 256" "512 1024 27 27 1 2 256" "1024 2048 13 13 1 2 256"; do
  for v in 0 1; do
    DCONV_DEBUG=1 python -c "
import sys; sys.path.insert(0, '.')
from paper_1809_10170_b200 import _abi
_abi.lib().dconv_cuda_set_ffma_variant($v)
sys.argv = ['one_layer.py'] + '$shp 2'.split()
exec(open('tools/one_layer.py').read())
" 2>&1 | sort | uniq -c | sort -rn | head -3
  done
done
