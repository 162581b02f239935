import json, sys
for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:
        print(p, "no json", e); continue
    print(p, f"ms/step {d['ms_per_step']:.2f} it {d.get('iterations')} spmv {d['roofline']['achieved']} GB/s ({d['roofline']['frac']}) "
          f"setup {d.get('setup_s', 0):.2f}s kernels {d.get('kernels')} e2e {d['e2e']['value']*1e3:.1f} ms launches {d.get('gpu_launches')}")
