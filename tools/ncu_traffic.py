"""DRAM traffic per launch of each kernel class from an ncu --set full report (for bench.py's
roofline "traffic" key): dram__bytes_read.sum + dram__bytes_write.sum, averaged over the captured
launches of a kernel; classes as eks_profile names them.

  python tools/ncu_traffic.py gpurun_out/x.ncu-rep "source note" > profiles/ncu_traffic_<name>.json
"""
import collections
import csv
import json
import re
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kclass(name):
    if name.startswith("k_spmm"):
        return "spmm"
    m = re.match(r"k_sweep<(\d+), (\d+), (\d+), (\d+), (\d+)(?:, (\d+))?>", name)
    if m:
        nq, nl, up = int(m.group(2)), int(m.group(3)), m.group(6)
        if up == "1":
            return "coef"  # the t = 64 Gram sweep
        if nq > 0 and nl > 0:
            return "upcoef"
        return "update" if nq > 0 else "coef"
    if name.startswith("k_upcoef"):
        return "upcoef"
    if name.startswith("k_gram_w"):
        return "coef"
    if name.startswith("k_apply"):
        return "apply"
    if name.startswith("k_chol"):
        return "chol"
    return "other"


def main(path, note):
    if path.endswith(".csv"):  # a raw-page export (ncu -i x.ncu-rep --page raw --csv)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    per_kernel = collections.defaultdict(list)
    for row in r[2:]:
        d = dict(zip(h, row))
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[m].replace(",", "")) * UNIT[u[h.index(m)]]
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("eks::", "").strip()
        per_kernel[name].append(b)
    kern = {k: sum(v) / len(v) for k, v in per_kernel.items()}
    cls = collections.defaultdict(list)
    for k, v in per_kernel.items():
        cls[kclass(k)].extend(v)
    print(json.dumps({"_source": note, "kernels": kern, "classes": {c: sum(v) / len(v) for c, v in cls.items()}},
                     indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else path)
