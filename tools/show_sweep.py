import json, sys
for l in open(sys.argv[1]):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print(d['lib'][:22].ljust(22), str(d.get('m', d.get('case'))).ljust(8), round(d['ms'], 3),
          d.get('boundary_frac', ''))
