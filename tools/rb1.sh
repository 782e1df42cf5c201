# batch-1 layer latency, compact split-K kernel vs unrolled
cd /root/repo
for shp in "64 64 58 58 3 1 1" "192 64 28 28 1 1 1" "96 128 30 30 3 1 1" "256 384 15 15 3 1 1" "480 192 14 14 1 1 1" "512 512 9 9 3 1 1"; do
  echo "$(python tools/one_layer.py $shp 5 | tail -1)   | unrolled: $(DCONV_NO_COMPACT=1 python tools/one_layer.py $shp 5 | tail -1 | cut -d: -f2)"
done
