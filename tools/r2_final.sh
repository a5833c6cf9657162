#!/bin/bash
# Final round-2 GPU refresh: build, all GPU tests, smoke, default bench line, the u16 bench line,
# the launch list, ncu --set full of the fp32 lookup, the u16 lookup and the phase-2 kNN
# (summarised on the box; the reports are deleted to stay under gpurun's 64 MiB copy-back).
cd "${GRAFT_REPO_ROOT:-.}"
OUT=gpurun_out/final; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo "build rc=$?" >> $OUT/build.log
timeout 3000 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench_default.log 2>&1
timeout 1200 python bench.py --lookup u16 > $OUT/bench_u16.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
cp profiles/traffic.json $OUT/traffic.json
R=/tmp/ncurep; mkdir -p $R
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $R/prof_lookup -f $CMD > $OUT/ncu_lookup.log 2>&1
python tools/ncu_summary.py full $R/prof_lookup.ncu-rep $OUT/r02_ncu_lookup_c3.txt --traffic $OUT/traffic.json --kernel lookup > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $R/prof_lookup_u16 -f $CMD --lookup u16 > $OUT/ncu_lookup_u16.log 2>&1
python tools/ncu_summary.py full $R/prof_lookup_u16.ncu-rep $OUT/r02_ncu_lookup_u16_c3.txt > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:knn_eseq -s 60 -c 1 -o $R/prof_knn -f $CMD > $OUT/ncu_knn.log 2>&1
python tools/ncu_summary.py full $R/prof_knn.ncu-rep $OUT/r02_ncu_knn_c3.txt --traffic $OUT/traffic.json --kernel ccm_knn > /dev/null 2>&1
cp $R/prof_lookup_u16.ncu-rep $OUT/ 2>/dev/null
du -sh $OUT
echo done
