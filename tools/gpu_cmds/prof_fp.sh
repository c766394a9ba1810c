for spec in "red3 36" "lazy3 36"; do
  set -- $spec
  timeout 600 python tools/prof_one.py $1 $2 > gpurun_out/plain_$1_$2.log 2>&1 || continue
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_ -c 1 -f -o gpurun_out/prof_r1f_$1$2 python tools/prof_one.py $1 $2 > gpurun_out/ncu_r1f_$1$2.log 2>&1
done
cat gpurun_out/plain_red3_36.log gpurun_out/plain_lazy3_36.log
