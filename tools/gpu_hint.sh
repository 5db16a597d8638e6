for H in 0 1 2 0; do QS_LD_HINT=$H timeout 600 python bench.py --no-circuits --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bh$H.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bh$H.json').read().strip().splitlines()[-1]); print('hint $H', round(d['value'],1), round(d['kernels']['U2']['gbs'],1), d['clocks']['sm_mhz'])"; done
