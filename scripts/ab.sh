#!/bin/bash
# A/B timing of library variants: bash scripts/ab.sh "<probe configs>" lib1.so lib2.so ...
# (each .so under paper_1010_4639_b200/_lib/; "default" = the in-tree build)
mkdir -p gpurun_out
CFGS="$1"; shift
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = default ]; then
    timeout 600 python scripts/probe.py $CFGS 2>&1
  else
    SPCG_LIB=paper_1010_4639_b200/_lib/$lib timeout 600 python scripts/probe.py $CFGS 2>&1
  fi
done
