python -c "
import time, torch
t=time.time()
import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import systems
c = FF.Context(systems.hh_ring(3), [1000]); t1=time.time()
c.init_group([-20.0,0,0,0,0]*3,[100.0,1,1,1,1]*3,1000,1,0,1); c.step(1,0.01); c.sync(); t2=time.time()
print('hh create %.2fs first step %.2fs'%(t1-t, t2-t1))
"
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -4
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"; done
