import sys, os, time, json
sys.path.insert(0, os.getcwd())
import paper_2507_05045_b200 as msb
from paper_2507_05045_b200.solver import native_solve
inst = msb.generate_instance(int(sys.argv[1]), 100, 1)
for r in range(int(sys.argv[2])):
    t0 = time.perf_counter()
    sols, st = native_solve(inst, "all", None, device=0)
    print(json.dumps({"rep": r, "wall": time.perf_counter() - t0, "dev_ms": st["dev_ms_total"], "hh": st["hash_hits"], "launches": st["kernel_launches"]}), flush=True)
