# round-2 final evidence: per-program table, launch list of the bench command, ncu of the fused launch
python tools/program_perf.py > gpurun_out/r02_programs_perf.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-scale-configs > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-scale-configs > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
python tools/ncu_pyramid.py > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused2 -s 2 -c 2 -o gpurun_out/r02_fused_c3 python tools/ncu_pyramid.py > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
