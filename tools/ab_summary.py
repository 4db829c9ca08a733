"""Summarise gpurun_out/ab_TAG.txt (tools/ab_probe.sh): cold median per config and variant."""
import collections
import json
import sys

res = collections.defaultdict(list)
var = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        var = line.split()[1]
    elif line.startswith("{"):
        d = json.loads(line)
        res[(json.dumps(d["cfg"]), var)].append(d["cold_us"])
cfgs = sorted({k[0] for k in res}, key=lambda c: c)
for c in cfgs:
    vs = sorted({k[1] for k in res})
    print(f"{c:48s} " + "  ".join(f"{v} " + " ".join("%.2f" % x for x in res.get((c, v), [])) for v in vs))
