"""Summarise an ncu --csv launch list: per (kernel, grid) share, avg us, DRAM GB/s."""
import collections, csv, re, sys

def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Grid Size")}
    K = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        d = K.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]})
        try:
            d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
    return K

def main(path, top=25, skip=("random_normal", "transpose", "fill_f32", "convert_copy")):
    K = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in K.values():
        if any(s in d["name"] for s in skip):
            continue
        nm = re.sub(r"\(.*", "", d["name"])[:56] + " " + d["grid"]
        a = agg[nm]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"kernels {sum(a[0] for a in agg.values())}  total {tot/1e6:.2f} ms")
    for nm, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{a[1]/tot*100:5.1f}% n={a[0]:5d} avg={a[1]/a[0]/1e3:8.1f}us dram={a[2]/a[0]/1e6:8.2f}MB "
              f"GB/s={a[2]/max(a[1],1):7.1f}  {nm}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
