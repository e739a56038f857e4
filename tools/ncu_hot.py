"""Top SASS lines by warp-stall samples of one kernel in an ncu report (source page).
    python tools/ncu_hot.py REPORT [N] [--regions K]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(r[iS]) for r in data)
    print("total samples", tot, "instructions", len(data))
    # stall totals
    st = {c: sum(int(r[hdr.index(c)]) for r in data) for c in cols}
    print({k: v for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v})
    if "--regions" in sys.argv:
        k = int(sys.argv[sys.argv.index("--regions") + 1])
        for a in range(0, len(data), k):
            s = sum(int(r[iS]) for r in data[a:a + k])
            ex = max(int(r[iE]) for r in data[a:a + k])
            print(f"{a:5d} {s:6d} {100*s/tot:5.1f}%  maxexec {ex:9d}  {data[a][1].strip()[:50]}")
        return
    for k, r in sorted(enumerate(data), key=lambda kr: -int(kr[1][iS]))[:n]:
        top = sorted(((int(r[hdr.index(c)]), c) for c in cols), reverse=True)[:2]
        print(k, r[1].strip()[:64], r[iS], r[iE], top)


if __name__ == "__main__":
    main()
