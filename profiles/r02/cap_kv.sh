ncu --set full --clock-control none --import-source on -k regex:kv_project -s 2 -c 1 -o gpurun_out/r02_kvproj python profiles/kvproj_time.py > gpurun_out/ncu_kv.log 2>&1; echo ncu=$?
