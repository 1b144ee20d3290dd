"""Code-size map of a kernel: per 2 KB block the dominant source lines.  Dev tool.
usage: code_map.py <lib.so> <mangled kernel>"""
import re, collections, subprocess, sys, tempfile, os, glob
so, fn = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [c for c in glob.glob(d + "/*.cubin") if os.path.basename(c).startswith("kernels.")][0]
lines = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur = "?"; blk = collections.defaultdict(list); n = 0
for l in lines[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2); continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        blk[int(m.group(1), 16) // 0x800].append(cur); n += 1
print("instructions", n, "bytes", 16 * n)
for b in sorted(blk):
    c = collections.Counter(blk[b])
    print(f"{b * 0x800:6x}", " ".join(f"{k}x{v}" for k, v in c.most_common(5)))
