"""Post-process an ncu CSV (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of the first solve_multi call's launches into the LU
traffic summary bench.py reports (profiles/r01_lu_traffic_<tag>.json).
usage: python tools/lu_traffic.py launches.csv out.json"""
import collections
import csv
import json
import sys

LU_KERNELS = ("assemble_kernel", "panel2_kernel", "swap_kernel", "linv_kernel", "zgemm_sub_tma", "perm_kernel",
              "init_kernel", "diag_inv128_kernel", "ozaki_gemm_kernel", "ozaki_split_a_kernel", "ozaki_split_b_kernel",
              "ozaki_colscale_kernel")
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path, out, n=4096, pencils=128):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rows.append(dict(zip(hdr, r)))
    by = collections.OrderedDict()
    for d in rows:
        by.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = (
            float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    launches = list(by.values())
    # the LU stage: from the first assemble to the first solve (permute_kernel)
    lu = []
    started = False
    for k in launches:
        if "assemble_kernel" in k["name"]:
            started = True
        if started and "permute_kernel" in k["name"]:
            break
        if started and any(s in k["name"] for s in LU_KERNELS):
            lu.append(k)
    byt = sum(k["dram__bytes_read.sum"][0] + k["dram__bytes_write.sum"][0] for k in lu)
    ms = sum(k["gpu__time_duration.sum"][0] * SCALE[k["gpu__time_duration.sum"][1]] for k in lu)
    per = collections.Counter()
    for k in lu:
        per[k["name"]] += k["dram__bytes_read.sum"][0] + k["dram__bytes_write.sum"][0]
    flops = pencils * 8.0 * n ** 3 / 3.0
    mn = 2.0 * 16.0 * n * n * pencils
    d = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum on bench.py, "
                   f"the first solve_multi call's kernels from assemble to the first solve ({path})",
         "launches": len(lu), "kernels": sorted({k["name"] for k in lu}), "lu_ms_serialised": ms,
         "lu_dram_bytes": byt, "lu_dram_bytes_by_kernel": dict(per), "lu_flops": flops,
         "lu_flop_per_dram_byte": flops / byt, "algorithmic_min_bytes": mn,
         "note": "the LU must read and write every pencil at least once (2 x 16 n^2 B per pencil)",
         "traffic_over_min": byt / mn}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in d.items() if k not in ("kernels", "lu_dram_bytes_by_kernel")}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
