# first-layer reader shapes of the configs (dense input)
cd /root/repo
for shp in "3 64 229 229 7 2 64" "3 64 229 229 7 2 256" "3 64 226 226 3 1 32" "3 96 227 227 11 4 1" "3 64 229 229 7 2 1" "3 64 226 226 3 1 1"; do
  python tools/one_layer.py $shp 3 first 2>&1 | tail -1
done
