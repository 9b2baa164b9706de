"""Top SASS instructions by warp-stall samples from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    i_src, i_s, i_ni = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Warp Stall Sampling (Not-issued Samples)")
    stall_cols = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_")]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(float(r[i_s] or 0) for r in body) or 1.0
    print(f"total samples {tot:.0f}")
    for k, r in enumerate(body):
        r.append(k)
    for r in sorted(body, key=lambda r: -float(r[i_s] or 0))[:int(top)]:
        st = sorted(((float(r[j] or 0), h[6:]) for j, h in stall_cols), reverse=True)[:3]
        print(f"{r[-1]:5d} {float(r[i_s]) / tot * 100:5.1f}%  {r[i_src].strip()[:60]:60s} " +
              " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0))


if __name__ == "__main__":
    main(*sys.argv[1:])
