# A/B within one GPU box: VARIANTS="name:ENV=val,ENV2=val name2:..." (ENV may be CASC_LIB_OVERRIDE)
for r in 1 2; do for spec in $VARIANTS; do
  name=${spec%%:*}; envs=${spec#*:}
  ( for kv in ${envs//,/ }; do [ "$kv" != "-" ] && export "$kv"; done
    timeout 300 python bench.py --config ${CFG:-E2} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$name.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));print('$name', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:(v['launches']//5,round(v['ms']/5,3)) for k,v in d['kernels'].items()})" )
done; done
