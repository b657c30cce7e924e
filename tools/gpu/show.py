import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).readline())
        print(f, 'value %.1f'%d['value'], 'ms %.2f'%d['ms_per_step'], 'pass', ['%.2f'%x for x in d['roofline']['pass_ms']], 'frac %.3f'%d['roofline']['frac'], 'step_frac %.3f'%d['roofline']['step_frac_of_peak'])
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-2000:])
