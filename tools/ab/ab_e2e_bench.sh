# cfg1 e2e A/B through bench.py's own e2e leg and tools/e2e_probe.py:
# lib_ab/libsvt_{a,b,c}.so (untracked builds) swapped into lib/, alternated
L=paper_2508_15229_b200/lib
for i in 1 2 3; do
 for v in a b c; do
  cp $L/../lib_ab/libsvt_$v.so $L/libsvt.so
  echo "$v$i bench $(python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"]), d["e2e"]["breakdown"]["decode_host_ms_per_step"])')"
  echo "$v$i probe $(python tools/e2e_probe.py 2>/dev/null)"
 done
done
cp $L/../lib_ab/libsvt_c.so $L/libsvt.so
