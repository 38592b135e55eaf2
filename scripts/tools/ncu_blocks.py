"""Group an ncu SASS source page (csv) into straight-line blocks and print the
hottest ones with their instruction mix and stall shares."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[idx[k]].replace(",", ""))
    except (KeyError, ValueError):
        return 0.0


tot_exec = sum(f(r, "Instructions Executed") for r in data)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
blocks, cur = [], None
for i, r in enumerate(data):
    src = r[idx["Source"]]
    op = (src.split()[1] if src.startswith("@") else src.split()[0]) if src.split() else "?"
    ex = f(r, "Instructions Executed")
    if cur and abs(ex - cur["exec"]) < 1e-6:
        cur["n"] += 1
        cur["ops"][op] += 1
        for k in ("samp", "wait", "ssb", "bar", "lsb"):
            cur[k] += f(r, {"samp": "Warp Stall Sampling (All Samples)", "wait": "stall_wait",
                            "ssb": "stall_short_sb", "bar": "stall_barrier",
                            "lsb": "stall_long_sb"}[k])
    else:
        if cur:
            blocks.append(cur)
        cur = {"start": i, "exec": ex, "n": 1, "thr": f(r, "Avg. Threads Executed"),
               "ops": collections.Counter({op: 1}),
               "samp": f(r, "Warp Stall Sampling (All Samples)"), "wait": f(r, "stall_wait"),
               "ssb": f(r, "stall_short_sb"), "bar": f(r, "stall_barrier"),
               "lsb": f(r, "stall_long_sb")}
blocks.append(cur)
print(f"warp-instructions {tot_exec:.0f}, stall samples {tot_s:.0f}")
for b in sorted(blocks, key=lambda b: -b["samp"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    print(f"@{b['start']} n={b['n']} exec={b['exec']:.0f} inst={100 * b['exec'] * b['n'] / tot_exec:.1f}% "
          f"samples={100 * b['samp'] / tot_s:.1f}% thr={b['thr']:.1f} wait={100 * b['wait'] / tot_s:.1f}% "
          f"short_sb={100 * b['ssb'] / tot_s:.1f}% long_sb={100 * b['lsb'] / tot_s:.1f}% barrier={100 * b['bar'] / tot_s:.1f}%")
    print("     ", b["ops"].most_common(10))
