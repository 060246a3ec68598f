#!/usr/bin/env python
"""Summarise a tools/ab.sh JSONL: per (shape, variant) the us/step of every round and the mean."""
import collections
import json
import sys

d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    j = json.loads(line)
    d[(j["shape"], j["variant"])].append(j["us_per_step"])
for (shape, var), v in sorted(d.items()):
    print(f"{shape:14s} {sum(v) / len(v):8.2f}  [{' '.join('%.2f' % x for x in v)}]  {var}")
