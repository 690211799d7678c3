"""Dev tool: top stall / instruction lines of an `ncu --page source --csv
--print-source sass` export (first kernel section by default)."""
import csv, sys

path = sys.argv[1]
sec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
s = sections[sec]
hdr, data = s["rows"][0], [r for r in s["rows"][1:] if len(s["rows"][0]) == len(r)]
ie, st, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
f = lambda x: float(x) if x not in ("", None) else 0.0  # noqa: E731
tot, tst = sum(f(r[ie]) for r in data), sum(f(r[st]) for r in data)
print(len(sections), "sections;", s["name"][:100])
print("warp instructions", tot, "stall samples", tst)
for r in sorted(data, key=lambda r: -f(r[st]))[:ntop]:
    print(r[0][-5:], r[st], r[ie], r[src][:100])
