"""DRAM bytes per launch of the z sweep (the bench's dominant kernel), averaged over the
launches of an ncu --set full capture of one RK4 step; writes profiles/sweep_dram_bytes.json
(read by bench.py for roofline.traffic).

    python tools/zsweep_dram.py gpurun_out/step.ncu-rep 512 > profiles/sweep_dram_bytes.json
"""
import csv
import io
import json
import subprocess
import sys


def main(path, n):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = []
    for r in rows[2:]:
        if r[ki].split("(")[0].replace("hd::", "").startswith("void sweep_kernel<2"):
            per.append(float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]])
    print(json.dumps({"kernel": "sweep_z", "n": n, "launches": len(per),
                      "bytes_per_launch": sum(per) / len(per), "per_launch": per,
                      "source": "ncu --set full, one fast-mode RK4 step at n^3 (tools/prof_step.py)"}))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
