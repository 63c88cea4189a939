"""Summaries of ncu outputs for profiles/ (run here, no GPU)."""
import csv, collections, json, subprocess, sys


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        try:
            v = float(r[iv].replace(",", ""))
        except (ValueError, IndexError):
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    out = {"launches": sum(cnt.values()), "total_ms": s / 1e6, "kernels": []}
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out["kernels"].append({"kernel": k, "launches": cnt[k], "ms": v / 1e6, "share": v / s})
    return out


def full_capture(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum"]
    caps = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        caps.append({k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k in keys})
    return caps


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    res = launch_list(path) if kind == "launches" else full_capture(path)
    print(json.dumps(res, indent=1))
