"""Check the repo's `file:line` citations into the reference (/root/reference/proj).

Every citation of the form ``name.cpp:A`` / ``name.hpp:A-B`` (also a bare
``:A-B`` continuing the last file named earlier in the same source file) is resolved against the
reference tree by basename.  A citation fails when
  * the cited range lies outside the file, or
  * an identifier that names a function defined in the cited file appears right
    before the citation (``symbol file.cpp:A-B`` / ``symbol :A-B``) and the
    cited range does not overlap that function's definition.

Usage: python tools/check_citations.py  (prints the failures, exit 1 if any).
Used by tests/test_citations.py.
"""
from __future__ import annotations

import os
import re
import sys

REF = "/root/reference/proj"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCAN_EXT = (".py", ".cu", ".cuh", ".cpp", ".h", ".hpp", ".md")
SKIP_FILES = {"SURVEY.md", "VERDICT.md", "BASELINE.md", "PAPERS.md", "SNIPPETS.md", "ADVICE.md"}
SKIP_DIRS = {".git", "gpurun_out", "_ref", "__pycache__", "build", "profiles", "golden", "bin"}

CITE = re.compile(r"(?:\b([A-Za-z_][\w]*\.(?:cpp|hpp|h)))?:(\d+)(?:-(\d+))?")
IDENT = re.compile(r"[A-Za-z_][\w:]*")


def ref_files():
    out = {}
    for d, _, fs in os.walk(REF):
        for f in fs:
            if f.endswith((".cpp", ".hpp", ".h")):
                out.setdefault(f, []).append(os.path.join(d, f))
    return out


def definitions(path):
    """name -> list of (first, last) line of each top-level definition (a line at
    column 0 containing `name(` whose body closes with a `}` at column 0)."""
    lines = open(path, encoding="utf-8", errors="replace").read().split("\n")
    defs = {}
    head = re.compile(r"^[A-Za-z].*?\b([A-Za-z_]\w*(?:::[A-Za-z_~]\w*)*)\s*\(")
    i = 0
    while i < len(lines):
        m = head.match(lines[i])
        if m and not lines[i].rstrip().endswith(";") and not lines[i].startswith(("return", "if", "for")):
            name = m.group(1).split("::")[-1]
            j = i
            while j < len(lines) and "{" not in lines[j] and not lines[j].rstrip().endswith(";"):
                j += 1
            if j < len(lines) and "{" in lines[j]:
                k = j
                if not (lines[j].rstrip().endswith("}") and lines[j].count("{") == lines[j].count("}")):
                    k = j + 1
                    while k < len(lines) and not lines[k].startswith("}"):
                        k += 1
                defs.setdefault(name, []).append((i + 1, k + 1))
                i = k + 1
                continue
        i += 1
    return defs, len(lines)


def scan_files():
    for d, dirs, fs in os.walk(ROOT):
        dirs[:] = [x for x in dirs if x not in SKIP_DIRS]
        for f in fs:
            if f.endswith(SCAN_EXT) and f not in SKIP_FILES and f != "check_citations.py":
                yield os.path.join(d, f)


def check():
    refs = ref_files()
    cache = {}
    failures, total = [], 0
    for path in scan_files():
        rel = os.path.relpath(path, ROOT)
        last = None  # a bare :N continues the last file named in this source file
        for ln, line in enumerate(open(path, encoding="utf-8", errors="replace"), 1):
            for m in CITE.finditer(line):
                fname, a, b = m.group(1), int(m.group(2)), int(m.group(3) or m.group(2))
                if fname:
                    last = fname
                elif last is None or m.start() == 0 or line[m.start() - 1] not in " (`":
                    continue  # a bare :N only continues a file named earlier on the line
                fname = fname or last
                if fname not in refs:
                    continue
                if len(refs[fname]) > 1:
                    continue  # ambiguous basename
                total += 1
                rpath = refs[fname][0]
                if rpath not in cache:
                    cache[rpath] = definitions(rpath)
                defs, nlines = cache[rpath]
                where = f"{rel}:{ln}: {fname}:{a}" + (f"-{b}" if b != a else "")
                if a < 1 or b < a or b > nlines:
                    failures.append(f"{where} outside the file ({nlines} lines)")
                    continue
                before = line[:m.start()].rstrip(" `(")
                words = IDENT.findall(before[-60:])
                sym = words[-1].split("::")[-1] if words else None
                dm = re.match(r"\s*(?:def|class)\s+(\w+)", line)
                if dm and dm.group(1) in defs and sym not in defs:
                    sym = dm.group(1)  # `def name(...):  # file.cpp:A-B`
                if fname and sym and sym.endswith((".cpp", ".hpp")):
                    continue
                if sym in defs:
                    spans = defs[sym]
                    if not any(lo <= b and a <= hi for lo, hi in spans):
                        failures.append(f"{where} does not overlap `{sym}` at "
                                        + ", ".join(f"{lo}-{hi}" for lo, hi in spans))
    return failures, total


if __name__ == "__main__":
    if not os.path.isdir(REF):
        print("reference tree absent; nothing to check")
        sys.exit(0)
    fails, total = check()
    for f in fails:
        print(f)
    print(f"{total} citations checked, {len(fails)} failures")
    sys.exit(1 if fails else 0)
