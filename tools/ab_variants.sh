#!/bin/bash
# A/B timing of compile-time experiment switches (GPU box):
#   bash tools/ab_variants.sh NAME1=DEF1,DEF2 NAME2= ...   (empty = no defines)
for spec in "$@"; do
  name=${spec%%=*}; defs=${spec#*=}
  python - "$name" "$defs" <<'PY'
import sys
from paper_2007_09884_b200 import build as b
name, defs = sys.argv[1], sys.argv[2]
b.build_variant(name, [d for d in defs.split(",") if d])
PY
  echo "== $name ($defs)"
  OPMM_LIB=build/variants/libopmm_$name.so python tools/time_kv.py 2>&1 | head -2; OPMM_LIB=build/variants/libopmm_$name.so python tools/time_setup.py
done
