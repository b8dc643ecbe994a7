#!/bin/bash
# usage (on a B200): LIBS="a.so b.so" bash scripts/ab_index.sh -- index-stage (memset, k_lists,
# k_index) and k_decode ms per config-2 variant, serial schedule, and the overlapped step
for L in ${LIBS}; do for S in serial overlap; do
GC_LIB=$L timeout 600 python bench.py --config ${CFG:-2} --sched $S --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --extra-configs none 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); pc=l['per_codec']
print('$S', '$L'.split('/')[-1], 'step %.4f'%l['ms_per_step'], 'sum_idx %.4f'%sum(v['index_ms'] for v in pc.values()), 'sum_dec %.4f'%sum(v['decode_kernel_ms'] for v in pc.values()), ' '.join('%s:%.4f'%(k,v['index_ms']) for k,v in pc.items()))"
done; done
