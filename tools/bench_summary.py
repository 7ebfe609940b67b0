import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
out=[("asum", d['roofline']['frac'], d['roofline']['isolated']['frac'])]
for k,v in d['suite'].items():
    r=v.get('roofline',{}); out.append((k, r.get('frac'), r.get('isolated',{}).get('frac')))
print(sys.argv[2], " ".join(f"{k}={a:.3f}/{b:.3f}" for k,a,b in out))
