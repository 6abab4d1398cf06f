# One full ncu capture of the tracker kernel; the report stays on the box
# (too large for the 64 MiB merge-back): summary JSON + raw-page CSV come back.
mkdir -p gpurun_out
R=/tmp/prof_${1}_${2}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track -c 1 -o $R python tools/one_path.py $1 $2 > gpurun_out/ncu_${1}_${2}.log 2>&1
python tools/ncu_summary.py $R.ncu-rep ${1}-${2} > gpurun_out/ncu_full_${1}_${2}.json
ncu -i $R.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${1}_${2}.csv 2>/dev/null
ncu -i $R.ncu-rep --page details --csv > gpurun_out/ncu_details_${1}_${2}.csv 2>/dev/null
ls -la $R.ncu-rep gpurun_out
