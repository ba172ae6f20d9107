"""Write profiles/traffic.json entries for one workload from ncu --set full captures (one launch each).

  python tools/traffic_json.py <workload> <units_per_launch> <run tag> K1_fourier_op=<rep> K2_gemm_tn=<rep> ...

bench.py attaches dram__bytes_read.sum + dram__bytes_write.sum of the DOMINANT kernel of the same
workload, scaled from these units to its own launch width (roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, r = rows[0], rows[1], rows[2]

    def val(key, unit_to_bytes=True):
        i = h.index(key)
        v = float(r[i].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
        return v * scale.get(u[i], 1.0)
    return dict(kernel=r[h.index("Kernel Name")].split("(")[0], read=val("dram__bytes_read.sum"),
                write=val("dram__bytes_write.sum"), us=val("gpu__time_duration.sum"))


def main():
    wl, units, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    ent = data.setdefault(wl, {})
    for kv in sys.argv[4:]:
        name, rep = kv.split("=", 1)
        m = metrics(rep)
        ent[name] = {"bytes_per_launch": m["read"] + m["write"], "read": m["read"], "write": m["write"],
                     "units_per_launch": units, "kernel": m["kernel"], "us_under_ncu": round(m["us"], 1),
                     "run": tag}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(ent, indent=1))


if __name__ == "__main__":
    main()
