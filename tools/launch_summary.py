"""Per-kernel share of device time from an ncu launch list (gpu__time_duration.sum CSV)."""
import csv, re, sys

def short(name):
    base = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0]
    base = re.sub(r"<.*", "", base)
    return base.split("::")[-1].replace("void ", "").strip()

def main(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    iu = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    agg = {}
    for r in rows[start:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            f = scale.get(r[iu], 1e-3) if iu is not None else 1e-3
            agg.setdefault(short(r[ik]), []).append(float(r[iv].replace(",", "")) * f)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print("| %s | %d | %.1f | %.1f | %.3f |" % (k, len(v), sum(v), sum(v) / len(v), sum(v) / tot))

if __name__ == "__main__":
    main(sys.argv[1])
