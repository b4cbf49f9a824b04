#!/bin/bash
# A/B timings of kernel variants on C4 (3 sweeps) and C5 (1 sweep)
run() { python tools/profile_case.py $1 $2 2 | python -c "
import sys,ast
for line in sys.stdin:
    name,_,it,_,st=line.split(' ',4)
    s=ast.literal_eval(st.strip())
    print(name,'sandwich GB/s',round(s['sandwich_bytes']/1e9/(s['sandwich_ms']/1e3)),'avg us',round(1e3*s['sandwich_ms']/s['sandwich_launches'],1),'env avg us',round(1e3*s['env_ms']/max(1,s['env_launches']),1), 'alg GB', round(s['alg_bytes_total']/1e9,1))
"; }
for cfg in "C4 3" "C5 1"; do
  echo "== $cfg rows+warm";   run $cfg
  echo "== $cfg rows cold";   QF_WARM=0 run $cfg
  echo "== $cfg tile";   QF_SANDWICH=tile run $cfg
done
