timeout 300 python bench.py --no-batch --no-cpu-baseline --no-global --steps 20 > gpurun_out/b_plain.log 2>&1
timeout 300 python -c "
import torch, sys, runpy; torch.cuda.init(); torch.cuda.mem_get_info()
sys.argv=['bench.py','--no-batch','--no-cpu-baseline','--no-global','--steps','20']
runpy.run_path('bench.py', run_name='__main__')" > gpurun_out/b_torch.log 2>&1
for f in b_plain b_torch; do python -c "
import json; d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]); print('$f', d['e2e']['ms_per_step'], d['e2e']['ms_mean'], d['e2e']['ms_steps'])"; done
