# A/B sweep of the L2 bulk-prefetch distance on the bench step
for pf in 0 148 444 888 1776 3552; do
  D2Q37_PF_BLOCKS=$pf timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-extras --no-cpu > gpurun_out/pf_$pf.log 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/pf_$pf.log').read().strip().splitlines()[-1]); print('pf=$pf', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done
for pf in 0 444 1776; do
  D2Q37_PF_BLOCKS=$pf timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-extras --no-cpu --layout soa > gpurun_out/pfs_$pf.log 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/pfs_$pf.log').read().strip().splitlines()[-1]); print('soa pf=$pf', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done
