"""Compare two sweep logs/JSONs row by row: python tools/sweep_cmp.py A B"""
import json
import sys


def load(p):
    try:
        return {(r["prec"], r["row"]): r for r in json.load(open(p))["rows"]}
    except Exception:
        return {(r["prec"], r["row"]): r for r in (json.loads(l) for l in open(p) if l.startswith("{"))}


a, b = load(sys.argv[1]), load(sys.argv[2])
for k in a:
    if k in b:
        ra, rb = a[k], b[k]
        print(f"{k[0]} {k[1]:44s} {ra['seconds']*1e3:9.3f} -> {rb['seconds']*1e3:9.3f} ms  roof {ra['roof_frac']:.3f} -> {rb['roof_frac']:.3f}"
              f"  {'' if rb['parity_ok'] else 'PARITY FAIL'}")
