"""Where are the local-memory accesses of a kernel (by source line)?  Dev tool."""
import re, collections, subprocess, sys, tempfile, os, glob
so, fn = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [c for c in glob.glob(d + "/*.cubin") if "kernels" in os.path.basename(c) and "sim_api" not in os.path.basename(c)][0]
lines = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur = "?"; c = collections.Counter(); n = 0
for l in lines[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        n += 1
    mm = re.search(r"\b(STL|LDL)(\.\w+)*\b", l)
    if mm:
        c[(cur, mm.group(1))] += 1
print("instructions", n)
for k, v in sorted(c.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(k, v)
