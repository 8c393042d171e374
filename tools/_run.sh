timeout 1200 python -m pytest tests/test_gpu_zoom.py -x -q 2>&1 | tail -2
python tools/zoom_time.py 30
timeout 1200 python tools/sweep.py --kinds zoom --precs f64 --out gpurun_out/r14_sweep_zoom64.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['prec'], r['row'], round(r['seconds']*1e3,3), 'ms', r['bound'], round(r['roof_frac'],3), 'ok' if r['parity_ok'] else 'PARITY FAIL')
"
