#!/bin/bash
# Sphere SFC comparison on config 3 (655,362 cells): 3-D Morton (default) vs Hilbert per cube face.
# Bench ms/step per kind, then ncu L2 hit rate / DRAM bytes / time of the slow and stage kernels.
python -m paper_2405_10505_b200.build > gpurun_out/build.log 2>&1 || exit 1
for sfc in morton hilbert_face; do
  FBLTS_SFC=$sfc timeout 600 python bench.py --config config3 --steps 50 --no-cpu-baseline --no-e2e --no-global \
      > gpurun_out/sfc_$sfc.log 2>&1
  grep '^{' gpurun_out/sfc_$sfc.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$sfc ms/step %.4f'%d['ms_per_step'], ' '.join('%s=%.4f'%(n,v['ms_per_step']) for n,v in sorted(k.items())))"
done
for sfc in morton hilbert_face; do
  FBLTS_SFC=$sfc timeout 300 python scripts/one_step.py config3 4 > gpurun_out/sfc_plain_$sfc.log 2>&1 &&
  FBLTS_SFC=$sfc timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none -k regex:"k_slow|k_stage|k_coarse_vel" -s 6 -c 12 --csv python scripts/one_step.py config3 4 \
     > gpurun_out/sfc_ncu_$sfc.csv 2> gpurun_out/sfc_ncu_$sfc.err
done
