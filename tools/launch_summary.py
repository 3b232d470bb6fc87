"""Per-kernel summary of an ncu launch list (tools/profile.sh CSV): launches, device time and
its share, DRAM bytes per launch (the roofline `traffic`), and the tensor path counted by ncu
(sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32: bf16 tcgen05 MMA ops) as TF/s per launch.
usage: python tools/launch_summary.py launches.csv [--json]"""
import csv
import json
import re
import sys

SCALE_T = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
SCALE_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    base = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0]
    base = re.sub(r"<.*", "", base)
    return base.split("::")[-1].replace("void ", "").strip()


def summarize(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, im, iu, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Value", "Metric Name", "Metric Unit", "ID"))
    launches = {}
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        rec = launches.setdefault(r[iid], {"kernel": short(r[ik])})
        v = float(r[iv].replace(",", "") or 0)
        m = r[im]
        if m == "gpu__time_duration.sum":
            rec["us"] = v * SCALE_T.get(r[iu], 1e-3)
        elif m.startswith("dram__bytes"):
            rec["bytes"] = rec.get("bytes", 0.0) + v * SCALE_B.get(r[iu], 1.0)
        elif m == "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum":
            rec["ops"] = v
        elif m.endswith("pct_of_peak_sustained_elapsed"):
            rec.setdefault("pct", {})[m.split(".")[0]] = v
    agg = {}
    for rec in launches.values():
        if "us" not in rec:
            continue
        a = agg.setdefault(rec["kernel"], {"n": 0, "us": 0.0, "bytes": 0.0, "ops": 0.0, "pct_ops": 0.0, "pct_cyc": 0.0})
        a["n"] += 1
        a["us"] += rec["us"]
        a["bytes"] += rec.get("bytes", 0.0)
        a["ops"] += rec.get("ops", 0.0)
        a["pct_ops"] += rec.get("pct", {}).get("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32", 0.0)
        a["pct_cyc"] += rec.get("pct", {}).get("sm__pipe_tensor_cycles_active", 0.0)
    return agg


def main(path, as_json=False):
    agg = summarize(path)
    tot = sum(a["us"] for a in agg.values())
    if as_json:
        print(json.dumps({k: {"launches": a["n"], "mean_us": a["us"] / a["n"], "dram_bytes_per_launch": a["bytes"] / a["n"],
                              "tensor_ops_per_launch": a["ops"] / a["n"], "share": a["us"] / tot}
                          for k, a in agg.items()}, indent=1))
        return
    print("| kernel | launches | mean us | share | DRAM MB / launch | tensor ops / launch | ncu TF/s | "
          "ncu tensor-op % of peak | ncu tensor-pipe cycles % |\n|---|---|---|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        n = a["n"]
        tf = a["ops"] / n / (a["us"] / n * 1e-6) / 1e12 if a["us"] else 0.0
        print("| %s | %d | %.1f | %.3f | %.1f | %.3g | %.0f | %.1f | %.1f |" % (
            k, n, a["us"] / n, a["us"] / tot, a["bytes"] / n / 1e6, a["ops"] / n, tf, a["pct_ops"] / n,
            a["pct_cyc"] / n))


if __name__ == "__main__":
    main(sys.argv[1], "--json" in sys.argv)
