"""Copy a tools/profile_round.sh run (gpurun_out/round) into profiles/:
bench lines, im2col comparison, ncu launch list, traffic.json."""
import glob
import json
import os
import shutil
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/round"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles"
for f in glob.glob(src + "/bench_*.log"):
    tag = os.path.basename(f)[6:-4]
    lines = [l for l in open(f) if l.startswith("{")]
    if not lines:
        print("no json line in", f)
        continue
    d = json.loads(lines[-1])
    name = {"reference": "r1_bench_reference_cpu.json"}.get(tag, f"r1_bench_{tag}.json")
    json.dump(d, open(os.path.join(dst, name), "w"), indent=1)
    print(name, d.get("value"))
for f in glob.glob(src + "/im2col_*.json"):
    shutil.copy(f, os.path.join(dst, "r1_" + os.path.basename(f).replace("im2col_", "im2col_vs_direct_")))
for a, b in (("launches_vgg16.csv", "r1_launches_vgg16_b32.csv"), ("nvidia_smi.txt", "r1_nvidia_smi.txt"),
             ("bench_default_wall.txt", "r1_bench_default_wall.txt"),
             ("launches_vgg16_tf32x3.csv", "r1_launches_vgg16_b32_tf32x3.csv")):
    if os.path.exists(os.path.join(src, a)):
        shutil.copy(os.path.join(src, a), os.path.join(dst, b))
full = json.load(open(os.path.join(dst, "r1_ncu_full_conv_ffma.json")))


def mb(s):
    v, u = s.split()
    return float(v) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[u]


t = json.load(open(os.path.join(dst, "traffic.json")))
for key, rep in (("vgg16", "vgg16_conv1_2_b32"), ("vgg16_conv4_2", "vgg16_conv4_2_b32")):
    if rep in full:
        r = full[rep]
        t[key]["dram_bytes"] = int(mb(r["dram__bytes_read.sum"]) + mb(r["dram__bytes_write.sum"]))
x3f = os.path.join(dst, "r1_ncu_full_conv_tf32x3.json")
if os.path.exists(x3f):
    r = json.load(open(x3f)).get("vgg16_conv4_2_b32")
    if r:
        # 512->512 3x3, 30x30 -> 28x28, batch 32: input + output + weights once
        alg = 4 * (32 * 512 * 30 * 30 + 32 * 512 * 28 * 28 + 512 * 512 * 9)
        t["vgg16_tf32x3"] = {
            "kernel": "conv_tf32x3_kernel on VGG conv4_2 (512->512, 30->28, batch 32), one launch",
            "dram_bytes": int(mb(r["dram__bytes_read.sum"]) + mb(r["dram__bytes_write.sum"])),
            "algorithmic_bytes": alg,
            "source": "profiles/r1_ncu_full_conv_tf32x3.json (ncu --set full)"}
json.dump(t, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
