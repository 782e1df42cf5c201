# ResNet c3 shape (64->256 1x1 + skip-add + ReLU, 56x56, b256): tile width sweep
cd /root/repo
for v in 0 1; do for tw in 8 16 28 32 56; do
  echo "variant $v TW $tw: $(DCONV_FORCE_TW=$tw python -c "
import sys; sys.path.insert(0, '.')
from paper_1809_10170_b200 import _abi
_abi.lib().dconv_cuda_set_ffma_variant($v)
sys.argv = ['one_layer.py'] + '64 256 56 56 1 1 256 3 ffma_add'.split()
exec(open('tools/one_layer.py').read())
" 2>&1 | tail -1)"
done; done
