"""Copy a tools/profile_round.sh run (gpurun_out/round) into profiles/:
bench lines and the DRAM traffic of the headline kernel (traffic.json).
usage: python tools/save_round.py [src] [dst] [tag]"""
import json
import os
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/round"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles"
tag = sys.argv[3] if len(sys.argv) > 3 else "r2"
names = {"bench_default.log": "bench_default", "bench_tf32x3.log": "bench_tf32x3",
         "bench_tf32.log": "bench_tf32", "bench_reference.log": "bench_reference_cpu",
         "bench_resnet50_co_nccl.log": "bench_resnet50_co_nccl",
         "bench_resnet50_co_peer.log": "bench_resnet50_co_peer"}
for f, n in names.items():
    p = os.path.join(src, f)
    if not os.path.exists(p):
        continue
    lines = [l for l in open(p) if l.startswith("{") and '"metric"' in l]
    if not lines:
        print("no json line in", p)
        continue
    d = json.loads(lines[-1])
    json.dump(d, open(os.path.join(dst, f"{tag}_{n}.json"), "w"), indent=1)
    print(f"{tag}_{n}.json", d.get("value"))
for f in ("bench_default_wall.txt", "nvidia_smi.txt", "launches_vgg16.csv",
          "launches_vgg16_tf32x3.csv"):
    p = os.path.join(src, f)
    if os.path.exists(p):
        open(os.path.join(dst, f"{tag}_{f}"), "w").write(open(p).read())


def mb(s):
    v, u = s.split()
    return float(v) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[u]


full = json.load(open(os.path.join(dst, f"{tag}_ncu_full_conv_ffma.json")))
t = json.load(open(os.path.join(dst, "traffic.json")))
r = full.get("vgg16_conv1_2_b32")
if r:
    t["vgg16"]["dram_bytes"] = int(mb(r["dram__bytes_read.sum"]) + mb(r["dram__bytes_write.sum"]))
    t["vgg16"]["source"] = (f"profiles/{tag}_ncu_full_conv_ffma.json (ncu --set full, "
                            "dram__bytes_read.sum + dram__bytes_write.sum); writes still "
                            "resident in L2 at kernel end are not counted by dram__bytes_write")
json.dump(t, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
print(json.dumps(t.get("vgg16"), indent=1))
