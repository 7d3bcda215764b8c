import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/probe.log'):
    if l.startswith('=='): print(l.strip()); continue
    if l.startswith('[spcg trace]'): print('   ', l.strip()[13:]); continue
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    if 'us_per_it' in d:
        print('  ', d['cfg'], d['iterations'], 'us/it %.2f' % d['us_per_it'], 'it/s %.0f' % d['it_per_s'],
              'frac %.3f' % d['it_frac'], 'spmv %.3f ms %.0f GB/s' % (d['spmv_ms'], d['spmv_GBs']))
