"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches, total and mean duration, share of the listed time.
Under ncu every launch is serialised and cold-cache: compare SHARES only."""
import collections, csv, sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14]
    hdr = rows[0]
    iN, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iU = hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        v = float(r[iV].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[iU], 1.0)
        agg[r[iN][:90]].append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    lines = ["%-90s %8s %12s %10s %7s" % ("kernel", "launches", "total_us", "mean_us", "share")]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append("%-90s %8d %12.1f %10.1f %6.1f%%" % (k, len(v), sum(v), sum(v) / len(v), 100 * sum(v) / tot))
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
