"""Map SASS of one kernel to source lines: code bytes and (optionally) ncu executed
instructions / stall samples per line.  Dev tool.
usage: sass_lines.py <nvdisasm -g output> <mangled kernel> [ncu source-page csv]"""
import csv, re, sys, collections
dis, fn = sys.argv[1], sys.argv[2]
lines = open(dis).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur = "?"
addr2src = {}
for l in lines[start + 1:]:
    if l.startswith("//----") or l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        addr2src[int(m.group(1), 16)] = cur
ex = collections.Counter(); st = collections.Counter(); ni = collections.Counter()
code = collections.Counter(addr2src.values())
if len(sys.argv) > 3:
    rows = list(csv.reader(open(sys.argv[3])))
    h = rows[1]; data = rows[2:]
    ia, ie, iss, ino = h.index("Address"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)"), h.index("stall_no_inst")
    base = int(data[0][ia], 16)
    for r in data:
        src = addr2src.get(int(r[ia], 16) - base, "?")
        ex[src] += int(r[ie]); st[src] += int(r[iss]); ni[src] += int(r[ino])
te = sum(ex.values()) or 1; ts = sum(st.values()) or 1
key = (lambda k: -st[k]) if len(sys.argv) > 3 else (lambda k: -code[k])
print(f"{'line':22s} {'bytes':>6s} {'exec%':>6s} {'samp%':>6s} {'noinst%':>7s}")
for k in sorted(code, key=key)[:int(sys.argv[4]) if len(sys.argv) > 4 else 60]:
    print(f"{k:22s} {code[k]*16:6d} {ex[k]/te*100:6.2f} {st[k]/ts*100:6.2f} {ni[k]/ts*100:7.2f}")
by_file = collections.Counter()
for k, c in code.items():
    by_file[k.split(":")[0]] += c * 16
print(dict(by_file))
