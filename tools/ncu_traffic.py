"""dram bytes per launch of one kernel in an ncu --set full report ->
profiles/select_main_ncu.json (bench.py's roofline.traffic).
python tools/ncu_traffic.py REPORT.ncu-rep OUT.json "capture description" """
import csv, io, json, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units, row = rows[0], rows[1], rows[2]


def val(key, scale):
    i = head.index(key)
    return float(row[i].replace(",", "")) * scale[units[i]]


B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
T = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
rd, wr = val("dram__bytes_read.sum", B), val("dram__bytes_write.sum", B)
rec = {"kernel": row[head.index("Kernel Name")].split("(")[0], "dram_bytes_read": int(rd),
       "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
       "gpu_time_us": round(val("gpu__time_duration.sum", T), 2), "capture": sys.argv[3] if len(sys.argv) > 3 else ""}
json.dump(rec, open(sys.argv[2], "w"), indent=2)
print(rec)
