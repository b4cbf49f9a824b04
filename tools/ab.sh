#!/bin/bash
# A/B timings of kernel variants: C4 (3 sweeps), C5 (1 sweep); resident vs stream
run() { python tools/profile_case.py $1 $2 2 | python -c "
import sys,ast
for line in sys.stdin:
    name,_,it,_,st=line.split(' ',4)
    s=ast.literal_eval(st.strip())
    ms = s['resident_ms'] if s['engine']==2 else s['sandwich_ms']
    print(name,'engine',s['engine'],'sandwich/resident ms',round(ms,2),'GB/s',round(s['sandwich_bytes']/1e9/(s['sandwich_ms']/1e3)) if s['sandwich_ms'] else '-','avg us',round(1e3*s['sandwich_ms']/max(1,s['sandwich_launches']),1),'env avg us',round(1e3*s['env_ms']/max(1,s['env_launches']),1), 'GFLOP/s', round(s['sweep_flops']/1e9/(ms/1e3)) if ms else '-')
"; }
for cfg in "C4 3" "C5 1"; do
  for k in reg rows tile; do
    echo "== $cfg stream $k";   QF_ENGINE=stream QF_SANDWICH=$k run $cfg
  done
done
echo "== C4 resident"; QF_ENGINE=resident run C4 3
