"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of
`bench.py --policy tiny --steps 1 --warmup 0 ...`: per-kernel time shares of the step, and
the share of euclidean_kernel at N = 8192 (the last 32 sweep points) for comparison with the
bench's `roofline.share_of_step` (ncu launches are cold and serialised: compare shares only).

    python scripts/launch_shares.py gpurun_out/launches.csv [points_per_n=32] [launches_per_point=5]
"""
import collections
import csv
import json
import sys


def main():
    path = sys.argv[1]
    ppn = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    lpp = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    rows, hdr = [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                rows.append((d["Kernel Name"].split("(")[0].replace("lscat::<unnamed>::", ""),
                             float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)))
    # the step starts at the first row_kernel launch (suite fills precede it)
    first = next(i for i, (k, _) in enumerate(rows) if "row_kernel" in k)
    step = rows[first:]
    tot = sum(t for _, t in step)
    by = collections.Counter()
    for k, t in step:
        by[k.split("<")[0]] += t
    rk = [t for k, t in step if "row_kernel" in k]
    n8192 = rk[-ppn * lpp:] if len(rk) >= ppn * lpp else []
    out = {"launches": len(step), "total_us": round(tot, 1),
           "share_by_kernel": {k: round(v / tot, 4) for k, v in by.most_common()},
           "euclid_n8192_share": round(sum(n8192) / tot, 4) if n8192 else None,
           "euclid_n8192_mean_us": round(sum(n8192) / len(n8192), 2) if n8192 else None}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
