import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        print(l.rstrip()); continue
    sw = {k[3:-3]: v for k, v in d.items() if k.startswith('tc_') and k.endswith('_us') and k != 'tc_us'}
    print(f"{d['model']:10s} {d['op']:8s} auto={d['auto']} tc={d['tc_us']}us {d['tc_tflops']}TF cublas={d['cublas_bf16_us']}us ratio={d['tc_over_cublas']}", sw)
