"""Tabulate a merge_variants JSON line (skips compiler noise before it)."""
import collections
import json
import re
import sys

text = open(sys.argv[1]).read()
d = json.loads(text[text.index('{"'):].strip().splitlines()[0])
rows = collections.defaultdict(dict)
for k, v in d.items():
    name, kk = k.rsplit("_k", 1)
    rows[name][int(kk)] = (v["us"], v["ok"])
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for n, r in rows.items():
    if pat and not pat.search(n):
        continue
    print("%-16s" % n, "  ".join("k%d %6.2f%s" % (kk, u, "" if ok else " BAD")
                                 for kk, (u, ok) in sorted(r.items())))
