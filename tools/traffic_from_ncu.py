"""profiles/traffic.json (bench.py `roofline.traffic`) from an ncu launch list
of the product NVTX range (tools/gpu_ncu_product.sh): DRAM read + write bytes
of one J^T W J p product = the sum over its kernels of the per-launch mean.

    python tools/traffic_from_ncu.py CONFIG LAUNCHES_CSV [PRODUCTS_IN_RANGE=2]
"""
import collections
import csv
import json
import os
import sys
import time


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    n_prod = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    for r in data:
        if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot[r[ki].split("(")[0]] += float(r[vi].replace(",", ""))
    per_product = sum(tot.values()) / n_prod
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    d = json.load(open(out_path)) if os.path.exists(out_path) else {}
    d[cfg] = int(per_product)
    d.setdefault("_source", {})[cfg] = {
        "launch_list": os.path.relpath(path), "products": n_prod,
        "kernels_bytes_per_product": {k: int(v / n_prod) for k, v in tot.items()},
        "written": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    json.dump(d, open(out_path, "w"), indent=1)
    print(cfg, per_product / 1e9, "GB per product")


if __name__ == "__main__":
    main()
