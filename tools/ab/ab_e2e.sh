# A/B of the cfg1 e2e line: lib_ab/libsvt_old.so vs lib_ab/libsvt_new.so (two
# builds made here from two source trees; not tracked) swapped into lib/ on the box
L=paper_2508_15229_b200/lib
for i in 1 2; do
 for v in old new; do
  cp $L/../lib_ab/libsvt_$v.so $L/libsvt.so
  timeout 400 python bench.py > gpurun_out/ab_$v$i.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v$i.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$v$i', round(d['value']), round(e['value']), round(e['breakdown']['prepare_ms_per_step'],3), round(e['breakdown']['decode_host_ms_per_step'],3))"
 done
done
