"""Summarise an A/B kbench log whose lines are '<tag>=<value> <case> <json>'."""
import collections
import json
import sys

d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    parts = line.split(" ", 2)
    if len(parts) < 3 or "=" not in parts[0]:
        print(line.rstrip())
        continue
    tag, name, js = parts
    try:
        d[(name, tag)].append(list(json.loads(js).values())[0]["us"])
    except (ValueError, KeyError, TypeError):
        continue
tags = sorted({k[1] for k in d})
for n in sorted({k[0] for k in d}):
    print(n, {t: d[(n, t)] for t in tags})
