"""One-line summary of a bench.py JSON line (used by the GPU scripts)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except (OSError, ValueError, IndexError) as e:
        print(path, "unreadable:", e)
        continue
    r = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    print(f"{d['config']['workload']:>9} {d['config'].get('path')} graph={d['config'].get('cuda_graph')} "
          f"ms/step={d['ms_per_step']:.3f} Mrows/s={d['value'] / 1e6:.2f} "
          f"dom={r.get('kernel')} frac={r.get('frac') or 0:.3f} step_frac={r.get('step_frac') or 0:.3f} "
          f"e2e={(e2e.get('value') or 0) / 1e6:.2f}M cpu={(cpu.get('value') or 0) / 1e6:.3f}M "
          f"launches={d.get('gpu_launches')} clocks={d.get('clocks', {}).get('sm_mhz')} "
          f"phases={ {k: round(v, 3) for k, v in (d.get('phases_ms_per_step') or {}).items()} }")
    t = d.get("tensor_path")
    if t:
        print(f"{'':>9} tensor path: ms/step={t['ms_per_step']:.3f} Mrows/s={t['value'] / 1e6:.2f} "
              f"phases={ {k: round(v, 3) for k, v in (t.get('phases_ms_per_step') or {}).items()} }")
