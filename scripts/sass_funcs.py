"""Aggregate ncu per-SASS instruction counts of k_step by source FUNCTION
(innermost inlined frame).  Dev tool.
usage: sass_funcs.py <nvdisasm -g dis> <mangled kernel> <ncu source csv (sass)> <n_veh>"""
import csv, re, sys, collections
dis, fn, csvp, nveh = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
SRC = {"kstep.cu": "paper_2406_10661_b200/csrc/kstep.cu", "model.cuh": "paper_2406_10661_b200/csrc/model.cuh"}
ranges = {}
for f, p in SRC.items():
    cur = "?"
    rs = []
    for i, l in enumerate(open(p).read().splitlines(), 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:static\s+)?__(?:device|global)__.*?\b(\w+)\s*\(", l)
        if m and not l.startswith(" "):
            cur = m.group(1)
        elif re.match(r"^\w.*\b(\w+)\(.*\)\s*\{\s*$", l) and not l.startswith(" "):
            cur = re.match(r"^\w.*?\b(\w+)\(", l).group(1)
        rs.append(cur)
    ranges[f] = rs
lines = open(dis).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur = "?"
a2s = {}
for l in lines[start + 1:]:
    if l.startswith("//----") or l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        f = m.group(1).split("/")[-1]
        ln = int(m.group(2))
        cur = f + ":" + (ranges[f][ln - 1] if f in ranges and ln <= len(ranges[f]) else str(ln))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        a2s[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvp)))
h = rows[1]; data = rows[2:]
ia, it, iss = h.index("Address"), h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
base = int(data[0][ia], 16)
th = collections.Counter(); st = collections.Counter(); wi = collections.Counter()
for r in data:
    s = a2s.get(int(r[ia], 16) - base, "?")
    th[s] += int(r[it]); st[s] += int(r[iss]); wi[s] += int(r[ie])
tt = sum(th.values()); ts = sum(st.values()); tw = sum(wi.values())
print(f"thread inst / vehicle {tt / nveh:.0f}; warp inst / vehicle {tw / nveh:.1f}")
for k, v in th.most_common(40):
    print(f"{k:40s} thr/veh {v / nveh:7.1f}  warp/veh {wi[k] / nveh:6.2f}  samples {st[k] / ts * 100:5.1f}%")
