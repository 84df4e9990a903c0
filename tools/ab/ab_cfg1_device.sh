# cfg1 device-rate A/B (bench.py without e2e / secondaries / cpu baseline):
# lib_ab/libsvt_old.so vs _new.so (untracked builds), alternated 3 times
L=paper_2508_15229_b200/lib
for i in 1 2 3; do
 for v in old new; do
  cp $L/../lib_ab/libsvt_$v.so $L/libsvt.so
  echo "$v$i $(python bench.py --no-secondary --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["avg_launch_us"],3), round(r["frac"],3), r["general_contract"]["us_per_token"], r["warm"]["us_per_token"])')"
 done
done
cp $L/../lib_ab/libsvt_new.so $L/libsvt.so
