#!/bin/bash
# A/B of exchange variants of the cluster engines: N flushed solves each
mkdir -p gpurun_out
N=${N:-40}
for lib in ${LIBS:-paper_1010_4639_b200/_lib/libspcg_b200.so}; do
  echo "== $lib"
  SPCG_LIB=$lib timeout 600 python scripts/bimodal.py $N ${CASES:-csr:6,sympriv:6,csc:6,sympriv:5,symatom:5,csr:5} | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['case'], 'min', d['us_it_min'], 'med', d['us_it_median'], 'mean', d['us_it_mean'], 'max', d['us_it_max'], 'slow', d['slow_runs'])"
done
