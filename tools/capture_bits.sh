# --set full of the bits-kernel launches of one re-plan (final build): the
# k = 16 launches of the bench re-plan, the k <= 8 ones of the forecast-like
# re-plan
ncu --set full --clock-control none --import-source on -k regex:hist_bits -c 4 -o gpurun_out/final_bits16 python tools/prof_replan.py --case bench --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:hist_bits -c 4 -o gpurun_out/final_bits8 python tools/prof_replan.py --case predict --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/final_bits16.ncu-rep > gpurun_out/final_ncu_bits16.txt 2>&1
ncu -i gpurun_out/final_bits8.ncu-rep > gpurun_out/final_ncu_bits8.txt 2>&1
rm -f gpurun_out/final_bits16.ncu-rep gpurun_out/final_bits8.ncu-rep
