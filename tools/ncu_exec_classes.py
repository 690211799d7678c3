"""Dev tool: group the SASS lines of an ncu source export by execution count
(lines of one loop body share it): instructions and stall samples per class."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
sec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
end = starts[sec + 1] if sec + 1 < len(starts) else len(rows)
hdr = rows[starts[sec] + 1]
data = [r for r in rows[starts[sec] + 2:end] if len(r) == len(hdr)]
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x) if x not in ("", None) else 0.0  # noqa: E731
by, bs, nl = collections.Counter(), collections.Counter(), collections.Counter()
for r in data:
    n = f(r[ie])
    k = round(n / 1e5) * 1e5
    by[k] += n
    bs[k] += f(r[st])
    nl[k] += 1
tot = sum(by.values())
print(rows[starts[sec]][1][:90], f"total {tot / 1e9:.3f}G")
for k, v in sorted(by.items(), key=lambda x: -x[1])[:20]:
    print(f"exec {k / 1e6:8.2f}M  lines {nl[k]:4d}  instr {v / 1e9:6.3f}G ({100 * v / tot:4.1f}%)  stalls {bs[k]:8.0f}")
