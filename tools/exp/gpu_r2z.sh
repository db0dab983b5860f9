mkdir -p gpurun_out
L=paper_2603_28845_b200/lib
for v in new base; do
  if [ $v = base ]; then cp $L/libocwg.so $L/libocwg_new.so; cp $L/libocwg_base.so $L/libocwg.so; fi
  for c in c3down c5down; do
    echo "== $v" >> gpurun_out/phases.log
    timeout 600 python tools/phases_cfg.py $c >> gpurun_out/phases.log 2>&1
  done
done
cp $L/libocwg_new.so $L/libocwg.so
