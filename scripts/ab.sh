#!/bin/bash
# A/B timing of library variants: scripts/ab.sh "<bench args>" lib1 lib2 ...
args="$1"; shift
for lib in "$@"; do
  echo "== $lib"
  GC_LIB=$lib timeout 300 python bench.py $args --no-e2e --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print('  total %.3f ms'%d['ms_per_step'], 'parity', d['parity']['verified'])
        for k,v in d['per_codec'].items(): print('   %-9s dec %.4f ms idx %.4f  %6.1f GB/s'%(k,v['decode_kernel_ms'],v['index_ms'],v['decode_kernel_gbs']))
    elif 'PARITY' in l or 'Error' in l: print('  ',l.strip()[:200])
"
done
