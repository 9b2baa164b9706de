"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the hot kernels from
ncu --set full captures → profiles/<tag>_traffic.json, read by bench.py's roofline "traffic" field."""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(out, *reps):
    res = {}
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
            b = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                b += float(d[k].replace(",", "")) * UNITS[units[hdr.index(k)]]
            dur = float(d["gpu__time_duration.sum"].replace(",", ""))
            dur *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[units[hdr.index("gpu__time_duration.sum")]]
            res[name] = {"dram_bytes_per_launch": b, "duration_us": dur,
                         "report": rep.split("/")[-1]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
