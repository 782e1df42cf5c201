#!/bin/bash
# A/B of build-free knobs on the VGG layers (variants 0 and 3)
for env in "X=1" "DCONV_FLUSH_EVERY=100000" "DCONV_RUNTIME_WF=1" "DCONV_FLUSH_EVERY=100000 DCONV_RUNTIME_WF=1"; do
  echo "== env: $env"
  env $env python tools/sweep_variants.py vgg16 32 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    try: d = json.loads(line)
    except Exception: print(line.strip()); continue
    print(d['layer'], d['tflops_by_variant']['0'], d['tflops_by_variant']['3'])
"
done
