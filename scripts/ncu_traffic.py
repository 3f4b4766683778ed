"""Record the DRAM traffic and warp execution efficiency of one `ncu --set
full` capture (one launch = one traversal) in profiles/ncu_traffic.json,
which bench.py reports as roofline.traffic / roofline.warp_efficiency.
Usage: python scripts/ncu_traffic.py <report.ncu-rep> "<bench workload key>" <summary path to cite>"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, key, cite):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, r = rows[0], rows[1], rows[2]

    def val(name):
        i = hdr.index(name)
        x = float(r[i].replace(",", ""))
        u = units[i].lower()
        return x * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    byts = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    weff = val("smsp__thread_inst_executed_per_inst_executed.ratio") / 32.0
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[key] = {"bytes_per_launch": byts, "warp_efficiency": weff,
              "source": "%s (ncu --set full, one launch = one traversal)" % cite}
    json.dump(d, open(path, "w"), indent=1)
    print(key, byts, weff)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
