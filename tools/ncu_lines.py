"""Per-source-line instruction and stall totals of one kernel in an ncu report
(run here): joins `--page source --print-source sass` metrics (per SASS
address) with the `cuda,sass` address -> source line map.

    python tools/ncu_lines.py <report.ncu-rep> [top]
"""
import collections
import csv
import io
import subprocess
import sys


def page(rep, src):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", src],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    sass = page(rep, "sass")
    hdr = sass[1]
    iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    met = {}
    for r in sass[2:]:
        try:
            met[int(r[0], 16)] = (float(r[iS]), float(r[iE]))
        except (ValueError, IndexError):
            pass
    addrs = sorted(met)
    mix = page(rep, "cuda,sass")
    owner = {}
    f, line, text, prev = "?", None, "", None
    for r in mix:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 4 or r[0] == "Line No":
            continue
        if r[0]:
            line, text, prev = (f, int(r[0])), r[1], None
            continue
        a = r[2]
        if a == "...":
            prev = ("range", prev)
            continue
        try:
            v = int(a, 16)
        except ValueError:
            continue
        if isinstance(prev, tuple) and prev[1] is not None:
            lo = prev[1]
            for x in addrs:
                if lo < x < v:
                    owner[x] = (line, text)
        owner[v] = (line, text)
        prev = v
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    for a, (s, e) in met.items():
        key, text = owner.get(a, (("?", 0), ""))
        agg[key][0] += s
        agg[key][1] += e
        agg[key][2] = text
    ts = sum(v[0] for v in agg.values())
    te = sum(v[1] for v in agg.values())
    print(f"total stall samples {ts:.0f}, warp instructions executed {te:.3e}")
    for key, (s, e, text) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{key[0]}:{key[1]:<5} instr {e / te * 100:5.1f}%  stalls {s / ts * 100:5.1f}%  {text[:80]}")


if __name__ == "__main__":
    main()
