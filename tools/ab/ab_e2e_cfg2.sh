# A/B of tools/e2e_probe_cfg2.py: lib_ab/libsvt_old.so vs lib_ab/libsvt_new.so
# (untracked builds) swapped into lib/ on the box, alternated 3 times
L=paper_2508_15229_b200/lib
for i in 1 2 3; do
 for v in old new; do
  cp $L/../lib_ab/libsvt_$v.so $L/libsvt.so
  echo "$v$i $(python tools/e2e_probe_cfg2.py 2>/dev/null)"
 done
done
