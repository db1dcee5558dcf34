"""Top stalled SASS instructions of each kernel in an ncu report (source page).

    python tools/ncu_top.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kernels, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            kernels.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None and r:
            cur[2].append(r)
    for name, h, d in kernels:
        i_s, i_src, i_a = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Address")
        tot = sum(int(r[i_s]) for r in d if r[i_s].isdigit()) or 1
        print(f"== {name[:100]}  samples {tot}")
        for r in sorted(d, key=lambda r: -int(r[i_s]) if r[i_s].isdigit() else 0)[:top]:
            print(f"{int(r[i_s]):7d} {100 * int(r[i_s]) / tot:5.1f}% {r[i_a][-5:]} {r[i_src].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
