"""Time one solve variant with CUDA events (diagnostics: join strategy / hash-only floor)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_05045_b200 as msb
from paper_2507_05045_b200 import _native
m, seed, flags, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
wave_keys = int(sys.argv[5]) if len(sys.argv) > 5 else 0
inst = msb.generate_instance(m, 100, seed)
opts = _native.make_options(mode="all", flags=flags | _native.MSP_FLAG_FORCE_TABLE_PATH, wave_keys=wave_keys)
best = None
for r in range(reps):
    rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
    assert rc in (0, 4), _native.last_error()
    best = st["dev_ms_total"] if best is None else min(best, st["dev_ms_total"])
print(json.dumps({"m": m, "flags": flags, "wave_keys": wave_keys, "best_dev_ms": best, "dev_ms_join": st["dev_ms_join"], "waves": st["waves"], "launches": st["kernel_launches"]}))
