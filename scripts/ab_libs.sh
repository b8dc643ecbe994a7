#!/bin/bash
# usage (on a B200, e.g. through gpurun): CFGS="2 4" LIBS="build/libgc_x.so paper_1502_01916_b200/libgc.so" bash scripts/ab_libs.sh
# A/B: bench per-variant decode times (and step) with several libraries: LIBS="a.so b.so"
for c in ${CFGS:-2 4}; do for L in ${LIBS}; do
GC_LIB=$L timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --extra-configs none 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); pc=l['per_codec']
print('$c', '$L'.split('/')[-1], 'step %.4f'%l['ms_per_step'], 'sum_dec %.4f'%sum(v['decode_kernel_ms'] for v in pc.values()), ' '.join('%s:%.4f'%(k,v['decode_kernel_ms']) for k,v in pc.items()))"
done; done
