"""Summarise an ncu launch-list CSV (--metrics ... --csv --log-file): per kernel the launch
count, average device time, share of the listed time and DRAM bytes per launch."""
import collections
import csv
import io
import sys


def summarise(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows:
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        agg[k][r["Metric Name"]] += v * scale
        if r["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        n = cnt[k]
        t = a["gpu__time_duration.sum"]
        out.append(f"{k:34s} launches={n:5d} avg={t / n:10.2f} us share={t / tot * 100:6.2f}% "
                   f"dram_rd/launch={a['dram__bytes_read.sum'] / n / 1e6:9.2f} MB "
                   f"dram_wr/launch={a['dram__bytes_write.sum'] / n / 1e6:8.2f} MB")
    return "\n".join(out) + f"\ntotal listed device time {tot / 1e3:.2f} ms over {sum(cnt.values())} launches"


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
