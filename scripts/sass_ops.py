"""Per-function SASS opcode counts of a kernel (dev tool).
usage: sass_ops.py <nvdisasm -g dis> <mangled kernel>"""
import re, sys, collections
dis, fn = sys.argv[1], sys.argv[2]
SRC = {"kstep.cu": "paper_2406_10661_b200/csrc/kstep.cu", "model.cuh": "paper_2406_10661_b200/csrc/model.cuh"}
ranges = {}
for f, p in SRC.items():
    cur = "?"; rs = []
    for l in open(p).read().splitlines():
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:static\s+)?__(?:device|global)__.*?\b(\w+)\s*\(", l)
        if m and not l.startswith(" "):
            cur = m.group(1)
        rs.append(cur)
    ranges[f] = rs
lines = open(dis).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur = "?"; c = collections.defaultdict(collections.Counter)
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        f = m.group(1).split("/")[-1]; ln = int(m.group(2))
        cur = f + ":" + (ranges[f][ln - 1] if f in ranges and ln <= len(ranges[f]) else str(ln)); continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", l)
    if m:
        c[cur][m.group(1)] += 1
tot = collections.Counter()
for k in c: tot.update(c[k])
print("TOTAL", {o: tot[o] for o in ("LD", "LDS", "LDG", "ST", "STS", "STG", "LDL", "STL")})
for k in sorted(c, key=lambda k: -sum(c[k].values()))[:25]:
    d = c[k]
    print(f"{k:32s} n={sum(d.values()):5d}", {o: d[o] for o in ("LD", "LDS", "LDG", "ST", "STS", "LDL", "STL") if d[o]})
