# A/B of the cfg2 split step (tools/time_static_half.py) and the static GEMM
# phase stamps (tools/cert_stamps.py): lib_ab/libsvt_old.so vs _new.so
# (untracked builds) swapped into lib/ on the box, alternated 3 times
L=paper_2508_15229_b200/lib
for i in 1 2 3; do
 for v in old new; do
  cp $L/../lib_ab/libsvt_$v.so $L/libsvt.so
  echo "$v$i $(python tools/time_static_half.py 2>/dev/null | tail -1)"
  [ $i = 1 ] && echo "$v$i stamps $(python tools/cert_stamps.py 2>/dev/null | tail -1)"
 done
done
cp $L/../lib_ab/libsvt_new.so $L/libsvt.so
