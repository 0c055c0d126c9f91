import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        try: d=json.loads(l)
        except Exception: print(l[:300]); continue
        print(d['lib'].split('/')[-1], {k:round(v['kernel_ms'],3) for k,v in d['res'].items()}, d['bitwise_equal_to_first'])
    elif not l.startswith('[gpurun] sending'): print(l.strip()[:200])
