# sweep K3 launch knobs on config 2: DS_SOLVE_RG (RHS per CTA), DS_SOLVE_NPC (packs per cluster)
for cfg in "0 8" "0 4" "0 2" "1 8" "2 8" "2 4" "4 4" "4 2" "8 1"; do
  set -- $cfg
  DS_SOLVE_RG=$1 DS_SOLVE_NPC=$2 timeout 100 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/sw.json 2>gpurun_out/sw_$1_$2.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('rg=$1 npc=$2', round(d['value'],1), 'RHS/s  solve ms/app', round(d['kernels']['block_solve']['ms_per_app'],2))" 2>/dev/null || echo "rg=$1 npc=$2 failed: $(tail -1 gpurun_out/sw_$1_$2.err)"
done
