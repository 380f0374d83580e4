#!/bin/bash
# A/B the Nelder-Mead kernel under compile-time switches (GPU box):
#   bash tools/ab_nm.sh NAME=DEF1,DEF2 ...
for spec in "$@"; do
  name=${spec%%=*}; defs=${spec#*=}
  python - "$name" "$defs" <<'PY'
import sys
from paper_2007_09884_b200 import build as b
b.build_variant(sys.argv[1], [d for d in sys.argv[2].split(",") if d])
PY
  echo "== $name ($defs)"
  OPMM_LIB=build/variants/libopmm_$name.so python tools/prof_nm.py 2048 2>&1 | tail -1
done
