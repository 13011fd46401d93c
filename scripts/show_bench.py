import json, sys
for p in sys.argv[1:]:
    for line in open(p):
        if line.startswith("{"):
            d = json.loads(line)
            k = d.get("kernels", {})
            print(p, "value=%.3f" % d["value"], "e2e=%s" % (d.get("e2e") or {}).get("value"),
                  " ".join("%s=%.4g" % (a, b) for a, b in k.items()),
                  "roof=%s" % {a: d["roofline"][a] for a in ("bound", "achieved", "frac")} if d.get("roofline") else "")
