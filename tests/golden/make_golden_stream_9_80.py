"""Batch headers (alpha, beta, n_left, n_right) of the reference stream at (9,80) s1 (TEST INFRASTRUCTURE).

oracle.stream_headers runs the heap enumeration of fastenum (restated in oracle/msp_oracle.c, pinned
to the reference's own streams in tests/test_oracle.py) over the full (9,80) instance: ~7 min on one
core.  The GPU's heap-free alpha plan must reproduce every header (tests/test_gpu_parity.py), and
make_golden_batches_9_80.py joins each batch on the CPU.

    python tests/golden/make_golden_stream_9_80.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2507_05045_b200.instances import generate_instance  # noqa: E402

if __name__ == "__main__":
    inst = generate_instance(9, 100, 1)
    hdrs = O.stream_headers(inst.a, inst.d)
    json.dump({"source": "oracle.stream_headers (heap stream restated from fastenum.py), generate_instance(9, 100, 1)",
               "columns": ["alpha", "beta", "n_left", "n_right"], "headers": [list(h) for h in hdrs]},
              open(os.path.join(HERE, "stream_9_100_1.json"), "w"), separators=(",", ":"))
    print(len(hdrs))
