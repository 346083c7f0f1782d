# Round-end ncu evidence for the default bench line (split schedule on C3): the launch list with
# DRAM bytes (-> profiles/traffic.json via tools/traffic_json.py) and one full capture of each
# split kernel (tree, emit) on 262,144 C3 roots.
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 --no-extra \
  > gpurun_out/ncu_launches_final.log 2>&1
for k in tree emit; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_${k}_kernel -s 1 -c 1 \
    -o /tmp/ncu/$k -f python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 --objects 262144 \
    > gpurun_out/ncu_${k}_final.log 2>&1
  ncu -i /tmp/ncu/$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_final_raw.csv 2>&1
  ncu -i /tmp/ncu/$k.ncu-rep --page source --csv > gpurun_out/ncu_${k}_source.csv 2>&1
  gzip -f gpurun_out/ncu_${k}_source.csv
done
