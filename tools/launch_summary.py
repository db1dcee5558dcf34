"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel+grid."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ix = {k: h.index(k) for k in ["ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit", "Metric Value"]}
    K = collections.defaultdict(dict)
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in data:
        v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
        K[int(r[ix["ID"]])].update({"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]],
                                    r[ix["Metric Name"]]: v})
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for v in K.values():
        t = v.get("gpu__time_duration.sum", 0.0)
        by = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
        a = agg[(v["name"][:70], v["grid"])]
        a[0] += 1
        a[1] += t
        a[2] += by
        tot += t
    print(f"launches {len(K)} total_us {tot:.1f} (ncu serialised, cold-cache)")
    for key, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{100 * a[1] / tot:6.2f}% n={a[0]:5d} avg_us={a[1] / a[0]:9.2f} "
              f"dramGB/s={a[2] / (a[1] * 1e3):7.1f} MB/launch={a[2] / a[0] / 1e6:8.2f} {key[1]:>14} {key[0]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
