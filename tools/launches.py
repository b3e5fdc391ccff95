"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per launch."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return data


if __name__ == "__main__":
    for (i, name), v in sorted(load(sys.argv[1]).items()):
        t = v.get("gpu__time_duration.sum", 0)
        rb, wb = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
        print(f"{i:3d} {name[:60]:60s} {t / 1e3:9.1f}us dram {(rb + wb) / max(t, 1):7.0f} GB/s rd {rb / 1e6:7.0f}MB wr {wb / 1e6:7.0f}MB")
