#!/bin/bash
# A/B of the two sandwich kernels on the bench config (C4, 3 sweeps) and C5 (1 sweep)
for cfg in "C4 3" "C5 1"; do
  for k in rows tile; do
    echo "== $cfg QF_SANDWICH=$k"
    QF_SANDWICH=$k python tools/profile_case.py $cfg 2 | python -c "
import sys,ast
for line in sys.stdin:
    name,_,it,_,st=line.split(' ',4)
    s=ast.literal_eval(st.strip())
    print(name,'sandwich GB/s',round(s['sandwich_bytes']/1e9/(s['sandwich_ms']/1e3)),'avg us',round(1e3*s['sandwich_ms']/s['sandwich_launches'],1),'env avg us',round(1e3*s['env_ms']/max(1,s['env_launches']),1))
"
  done
done
