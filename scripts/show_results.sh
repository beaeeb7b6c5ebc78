#!/bin/bash
# Summarise the last scripts/gpu_check.sh run (run from anywhere).
cd /root/repo
tail -2 gpurun_out/pytest_gpu.log
for f in bench_cfg2 bench_cfg3 bench_cfg1; do
  echo "== $f"
  python -c "
import json
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('value %.3e ms/step %.3f e2e %.3e' % (d['value'], d['ms_per_step'], d['e2e']['value']))
r=d['roofline']; print('map avg ms', r['avg_launch_ms'], 'share', r['share_of_device_time'], 'frac', r['frac'], 'tile_steps/s %.3e'%r['tile_steps_per_s'])
" 2>&1 | tail -2
done
[ -f gpurun_out/prof_cfg3.ncu-rep ] && python scripts/summarize_ncu.py full gpurun_out/prof_cfg3.ncu-rep | grep -E "Duration|Registers|Occupancy|Issue Slots|pipe_alu|hot loop|opcode|barrier|wait "
