# ncu captures of the final build: issue / pipe / DRAM metrics over every
# histogram launch (bench and forecast-like re-plans), and one --set full
# capture of each dominant kernel (row kernel stage-0 launch, bits kernel).
M=smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:hist_ --csv python tools/prof_replan.py --case bench --reps 2 > gpurun_out/final_metrics_bench.csv 2>&1
ncu --metrics $M --clock-control none -k regex:hist_ --csv python tools/prof_replan.py --case predict --reps 2 > gpurun_out/final_metrics_predict.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hist_rows_kernel" -c 1 -o gpurun_out/final_rows python tools/prof_replan.py --case bench --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hist_bits_kernel" -c 1 -o gpurun_out/final_bits python tools/prof_replan.py --case bench --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/final_rows.ncu-rep > gpurun_out/final_ncu_rows.txt 2>&1
ncu -i gpurun_out/final_bits.ncu-rep > gpurun_out/final_ncu_bits.txt 2>&1
rm -f gpurun_out/final_rows.ncu-rep gpurun_out/final_bits.ncu-rep
