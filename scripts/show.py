import json, sys, glob
for f in sys.argv[1:]:
    try: d=json.load(open(f))
    except Exception as e: print(f, e); continue
    print(f, 'ms/step', round(d['ms_per_step'],2), 'value', round(d['value'],2), 'roof', round(d['roofline']['frac'],3), 'k_ms', round(d['roofline']['avg_launch_ms'],3), 'resid', d.get('residual_after_cycle'))
    for k,v in d.get('breakdown',{}).items(): print('   ', k, round(v['ms_per_step'],3), v['launches_per_step'])
