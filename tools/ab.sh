#!/bin/bash
# A/B timings of kernel variants: C4 (3 sweeps), C5 (1 sweep); resident vs stream on C4/C3
run() { python tools/profile_case.py $1 $2 2 | python -c "
import sys,ast
for line in sys.stdin:
    name,_,it,_,st=line.split(' ',4)
    s=ast.literal_eval(st.strip())
    ms = s['resident_ms'] if s['engine']==2 else s['sandwich_ms']
    print(name,'engine',s['engine'],'sandwich/resident ms',round(ms,2),'GB/s',round(s['sandwich_bytes']/1e9/(s['sandwich_ms']/1e3)) if s['sandwich_ms'] else '-','avg us',round(1e3*s['sandwich_ms']/max(1,s['sandwich_launches']),1),'env avg us',round(1e3*s['env_ms']/max(1,s['env_launches']),1), 'GFLOP/s', round(s['sweep_flops']/1e9/(ms/1e3)) if ms else '-')
"; }
for cfg in "C4 3" "C5 1"; do
  echo "== $cfg stream rows";   QF_ENGINE=stream run $cfg
  echo "== $cfg stream tile";   QF_ENGINE=stream QF_SANDWICH=tile run $cfg
done
for cfg in "C4 3" "C3 20" "C2 50"; do
  echo "== $cfg resident";   QF_ENGINE=resident run $cfg
  echo "== $cfg stream";   QF_ENGINE=stream run $cfg
done
