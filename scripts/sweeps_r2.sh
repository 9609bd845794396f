# Round-2 sensitivity sweeps with the reference CSV schema (tools/dilithium_cli.cpp:448-514)
set -e
mkdir -p gpurun_out
for lv in 2 3 5; do
  tools/dilithium_b200 sweep --level $lv --phi 100000 --reps 5 --psi-min 12500 --psi-max 100000 --psi-steps 8 --streams-max 16 > gpurun_out/r02_sweep_level$lv.csv
  tools/dilithium_b200 sweep --level $lv --phi 10000 --reps 7 --psi-min 1250 --psi-max 10000 --psi-steps 8 --streams-max 8 | tail -n +2 >> gpurun_out/r02_sweep_level$lv.csv
done
head -40 gpurun_out/r02_sweep_level2.csv
