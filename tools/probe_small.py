import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import synth
from parity import run_parity
for name, b, s, m in [("C2",1,2,True),("C2",1,2,False),("C2",3,2,True),("C2",8,2,True),("C2",16,2,True),("C1",1,2,True),("C1",1,3,False),("C2",1,4,True),("C2",2,2,True)]:
    cfg = synth.CONFIGS[name].with_(seq=s)
    try:
        recs = run_parity(cfg, b, 1, steps=1, mixed=m)
        r = recs[0]
        print(name, b, s, m, "loss", r["loss_gpu"], r["loss_ref"], {k: round(v, 4) for k, v in r["grad_err"][0].items()}, flush=True)
    except Exception as e:
        print(name, b, s, m, "EXC", e, flush=True)
