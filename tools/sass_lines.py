"""Static SASS instructions per CUDA source line of one kernel (nvdisasm -g on the
extracted cubin).  usage: tools/sass_lines.py LIB.so CUBIN_NAME MANGLED_SUBSTRING [top]"""
import collections, os, re, subprocess, sys, tempfile

lib, cub, name = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
i = next(m.start() for m in re.finditer(r"^\.text\.(\S+):", txt, re.M) if name in m.group(1))
j = txt.find(".section", i + 10)
cur, cnt, ops = None, collections.Counter(), collections.defaultdict(collections.Counter)
for l in txt[i:j].split("\n"):
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
    if m and cur:
        op = m.group(2).split(".")[0]
        cnt[cur] += 1
        ops[cur][op] += 1
print("total", sum(cnt.values()))
for k, v in cnt.most_common(top):
    print(v, k, dict(ops[k].most_common(6)))
