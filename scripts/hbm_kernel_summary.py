"""Summarise an ncu CSV launch list of the HBM/latency-bound kernels
(k_split, k_compact_*, k_init, k_finalize, ...): per kernel the mean launch
time, DRAM bytes per launch and achieved DRAM GB/s against MEASURED_PEAKS.

  python scripts/hbm_kernel_summary.py gpurun_out/hbm_kernels.csv [out.json]
"""
import collections
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "%": 1, "": 1}


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    launches = collections.OrderedDict()
    for r in rows:
        if len(r) != len(hdr) or r == hdr:
            continue
        d = dict(zip(hdr, r))
        m = launches.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", "")})
        m[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1)
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs")
    agg = collections.defaultdict(list)
    for m in launches.values():
        agg[m["name"]].append(m)
    res = {}
    for k, ms in agg.items():
        t = sum(m["gpu__time_duration.sum"] for m in ms)
        b = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms)
        big = max(ms, key=lambda m: m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
        bb = big["dram__bytes_read.sum"] + big["dram__bytes_write.sum"]
        res[k] = {"launches": len(ms), "ms_per_launch": t / len(ms) * 1e3,
                  "dram_mb_per_launch": b / len(ms) / 1e6, "avg_dram_gbs": b / t / 1e9,
                  "largest_launch": {"grid": big.get("launch__grid_size"), "us": big["gpu__time_duration.sum"] * 1e6,
                                     "dram_mb": bb / 1e6,
                                     "dram_gbs": bb / big["gpu__time_duration.sum"] / 1e9,
                                     "dram_pct_of_peak_elapsed": big.get("dram__throughput.avg.pct_of_peak_sustained_elapsed")},
                  "hbm_peak_gbs": hbm}
    for k, v in sorted(res.items(), key=lambda x: -x[1]["ms_per_launch"] * x[1]["launches"]):
        g = v["largest_launch"]
        print(f"{k[:58]:58s} n={v['launches']:3d} {v['ms_per_launch']*1e3:8.1f} us/launch "
              f"{v['dram_mb_per_launch']:7.2f} MB  avg {v['avg_dram_gbs']:6.0f} GB/s | largest: "
              f"{g['us']:7.1f} us {g['dram_mb']:7.2f} MB {g['dram_gbs']:6.0f} GB/s grid {g['grid']}")
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
