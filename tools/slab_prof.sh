mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slabprof_cfg3_r8.csv python tools/slab_profile.py cfg3 8 3 > gpurun_out/slabprof.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slabprof_cfg3_r1.csv python tools/slab_profile.py cfg3 1 3 >> gpurun_out/slabprof.log 2>&1
tail -3 gpurun_out/slabprof.log
