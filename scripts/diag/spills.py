"""Where a kernel's local-memory spills sit: python scripts/diag/spills.py CUBIN NAME_SUBSTRING
(nvdisasm -g line info; counts STL/LDL per source line)."""
import collections, re, subprocess, sys
cubin, name = sys.argv[1], sys.argv[2]
out = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(out) if ".text." in l and name in l and "section" in l)
end = next((j for j in range(start + 1, len(out)) if ".section" in out[j] and ".text." in out[j]), len(out))
loc, cnt = None, collections.Counter()
for l in out[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        loc = (m.group(1).split("/")[-1], int(m.group(2)))
    if re.search(r"\b(STL|LDL)(\.\w+)*\b", l):
        cnt[loc] += 1
for k, v in sorted(cnt.items(), key=lambda kv: (str(kv[0][0]), kv[0][1])):
    print(f"{v:4d}  {k[0]}:{k[1]}")
print("total", sum(cnt.values()))
