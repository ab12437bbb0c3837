"""Markdown table of a directory of bench.py JSON lines (one file per config/precision):
workload, precision, dominant-kernel time, step, samples/s, roofline fraction, e2e, clock.

    python tools/sweep_table.py profiles/round2/final
"""
import glob
import json
import os
import sys


def line(path):
    with open(path) as f:
        for ln in reversed(f.read().strip().splitlines()):
            if ln.startswith("{"):
                return json.loads(ln)
    return None


def fmt_t(ms):
    return "%.1f µs" % (ms * 1e3) if ms < 0.1 else "%.3f ms" % ms if ms < 1 else "%.2f ms" % ms


def main(d):
    print("| file | workload | prec | mode | kernel | kernel time | step | samples/s | frac (bound) | path ceiling | e2e samples/s | SM MHz |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p in sorted(glob.glob(os.path.join(d, "*.json"))):
        x = line(p)
        if not x or "roofline" not in x:
            if x and x.get("impl") == "reference":
                print("| %s | %s | oracle f64 | — | — | — | %s | %.0f | — | — | — | — |" % (
                    os.path.basename(p), x["config"].get("workload"), fmt_t(x["ms_per_step"]), x["value"]))
            continue
        r, c = x["roofline"], x["config"]
        e2e = (x.get("e2e") or {}).get("value")
        print("| %s | %s | %s | %s | %s | %s | %s | %.3g | %.3f (%s) | %s | %s | %s |" % (
            os.path.basename(p), c.get("workload"), c.get("prec"), c.get("mode"), r.get("kernel"),
            fmt_t(r["kernel_ms"]), fmt_t(x["ms_per_step"]), x["value"], r["frac"], r["bound"],
            ("%.2f" % r["frac_of_path_ceiling"]) if "frac_of_path_ceiling" in r else "—",
            ("%.3g" % e2e) if e2e else "—", (x.get("clocks") or {}).get("sm_mhz")))


if __name__ == "__main__":
    main(sys.argv[1])
