for mode in cluster staged; do for g in 1 2; do
  if [ $mode = staged ]; then export DS_SOLVE_MODE=staged; else unset DS_SOLVE_MODE; fi
  DS_RHS_GROUPS=$g timeout 600 python bench.py --steps 3 --warmup 3 --config 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_$mode$g.json 2> gpurun_out/b3_$mode$g.err
  python -c "
import json; d=json.loads(open('gpurun_out/b3_$mode$g.json').read().strip().splitlines()[-1])
print('$mode groups $g', round(d['value'],2), round(d['roofline']['achieved'],2), round(d['kernels']['block_solve']['ms_per_app'],1))" || tail -3 gpurun_out/b3_$mode$g.err
done; done
