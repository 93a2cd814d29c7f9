import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l); L = d['line']
    print(f"{d['cfg']:8s} {d['kernel']:12s} {d['sigma0']:10s} rc={d['rc']}", end=' ')
    if L:
        print(f"{L['value']:.3e} samples/s ms {L['ms_per_step']:.3f} frac {L['roofline']['frac']:.3f} "
              f"{L['roofline']['bound']} {L.get('plan')}")
    else:
        print()
