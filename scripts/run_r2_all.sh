# End-of-change evidence run: GPU tests, bench line, ncu tables, launch list.  gpurun -- 'bash scripts/run_r2_all.sh'
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/${T:-r02}_gpu_tests.txt
cat gpurun_out/${T:-r02}_gpu_tests.txt
python bench.py > gpurun_out/${T:-r02}_bench.json 2> gpurun_out/${T:-r02}_bench.err || tail -5 gpurun_out/${T:-r02}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T:-r02}_bench_reference.json 2>> gpurun_out/${T:-r02}_bench.err
T=${T:-r02} bash scripts/run_r2_prof.sh 2>&1 | tail -5
