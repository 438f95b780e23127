mkdir -p gpurun_out
python tools/ncu_rounds.py > gpurun_out/nr_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rounds -s 6 -c 3 -o gpurun_out/nr_rounds_bulk -f python tools/ncu_rounds.py > gpurun_out/nr_ncu.log 2>&1
ncu -i gpurun_out/nr_rounds_bulk.ncu-rep --page raw --csv > gpurun_out/nr_rounds_bulk_raw.csv 2>/dev/null
ncu -i gpurun_out/nr_rounds_bulk.ncu-rep --page details --csv > gpurun_out/nr_rounds_bulk_details.csv 2>/dev/null
tail -n 5 gpurun_out/nr_plain.log; tail -n 3 gpurun_out/nr_ncu.log
