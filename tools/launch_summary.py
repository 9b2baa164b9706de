"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)
            out.append((d["Kernel Name"].split("(")[0].replace("void ", ""), v))
    return out


def main(path, last=None):
    ls = load(path)
    if last:
        ls = ls[-int(last):]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v in ls:
        tot[n] += v
        cnt[n] += 1
    T = sum(tot.values())
    print(f"{len(ls)} launches, {T / 1e3:.3f} ms total")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"  {k[:58]:58s} {cnt[k]:6d}  {v / 1e3:9.3f} ms  {v / cnt[k]:9.2f} us/launch  {100 * v / T:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
