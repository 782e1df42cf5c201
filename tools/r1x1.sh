cd /root/repo
for shp in "256 64 56 56 1 1 256" "64 64 56 56 1 1 256" "64 256 56 56 1 1 256" "128 512 28 28 1 1 256" "512 128 28 28 1 1 256" "1024 256 14 14 1 1 256"; do
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
