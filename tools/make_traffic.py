"""Write profiles/traffic.json: DRAM bytes (read + write) per launch of each library kernel, from an
ncu launch-list CSV of `bench.py --steps 1 --warmup 1` (the last step's launches are used).

    python tools/make_traffic.py gpurun_out/launches_TAG.csv CONFIG [WORLD]
"""
import csv
import json
import os
import sys
from collections import OrderedDict

NAMES = [("k_node_gather_t", "node_gather"), ("k_elem_scatter", "elem_scatter"), ("k_elem_segsort", "elem_segsort"),
         ("k_elem_count", "elem_count"), ("k_node_compact", "node_compact"), ("k_scan_i32", "scan_counts"),
         ("k_hist_validate", "hist_validate"), ("k_node_giant", "node_giant"), ("k_segsort_giant", "segsort_giant"),
         ("k_locality_sample", "locality_sample"), ("k_bucket_bases", "bucket_bases"),
         ("k_poly_count", "poly_count"), ("k_poly_scatter", "poly_scatter"), ("k_poly_gather", "poly_gather"),
         ("k_poly_giant", "poly_giant"), ("k_chunk_count", "count_fallback"), ("k_chunk_scatter<", "scatter_fallback"),
         ("k_chunk_scatter_fixed", "elem_scatter"),
         ("k_chunk_sort", "elem_segsort"), ("k_small_both", "small_both")]


def main():
    path, cfg = sys.argv[1], int(sys.argv[2])
    world = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    k = OrderedDict()
    for r in data:
        k.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    per = {}
    for (i, n), m in k.items():
        if "mn::" not in n:
            continue
        name = None
        if "k_onesweep" in n:
            # onesweep instances: <KeyT, SRC, T, PAYLOAD, OWNER, BINS, ..., RANK, COUNTS, EARLY>
            args = n[n.index("<") + 1:n.index(">")].split(",")
            src, payload, counts = int(args[1]), args[3].strip() in ("1", "true"), args[-2].strip() in ("1", "true")
            name = "onesweep_elem_first" if src == 2 else ("onesweep_elem_last" if counts else
                                                          ("onesweep_elem" if payload else "onesweep_node"))
        else:
            for key, nm in NAMES:
                if key in n:
                    name = nm
        if name is None:
            continue
        per.setdefault(name, []).append(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for name, vals in per.items():
        data[f"config{cfg}/n{world}/{name}"] = vals[-1]       # last (warm) launch
    data["_source"] = f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({os.path.basename(path)})"
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps({k: v for k, v in data.items() if k.startswith(f'config{cfg}/')}, indent=1))


if __name__ == "__main__":
    main()
