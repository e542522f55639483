#!/bin/bash
# scratch helper: (7,60) timing under env-variable settings given as arguments ("K=V K=V" per run)
for cfg in "$@"; do
  echo -n "$cfg  "
  env $cfg timeout 300 python tools/diag_time.py 7 1 0 3
done
