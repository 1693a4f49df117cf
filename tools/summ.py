"""One-line summary of a bench.py JSON line (stage times, a6 passes, roofline)."""
import json
import sys

for p in sys.argv[1:]:
    try:
        j = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable:", e)
        continue
    st = {k: round(v, 3) for k, v in j.get("stage_ms", {}).items()}
    r = j.get("roofline") or {}
    print(f"{j['config']['workload']}: {j['ms_per_step']:.3f} ms  {st}  roof {r.get('bound')} {r.get('frac', 0):.3f}"
          f"{'  parity ' + str({k: j['parity'][k] for k in ('mismatch', 'e_tok', 'e_elt')}) if j.get('parity') else ''}")
