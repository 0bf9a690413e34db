# ncu --set full with source counters for the group-by and the C4 index build; exports the raw
# page and the SASS-level source pages (per-instruction stall samples) as CSV.
python tools/profile_r2.py --ops groupby_c3,index_c4 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off \
    -o /tmp/src_prof python tools/profile_r2.py --ops groupby_c3,index_c4 > gpurun_out/src_prof.log 2>&1
ncu -i /tmp/src_prof.ncu-rep --page raw --csv > gpurun_out/src_prof_raw.csv
ncu -i /tmp/src_prof.ncu-rep --page source --csv --print-source sass -k regex:"k_aggregate<8" > gpurun_out/src_agg_sass.csv 2>&1
ncu -i /tmp/src_prof.ncu-rep --page source --csv --print-source sass -k regex:"k_histogram_seeded" > gpurun_out/src_hist_sass.csv 2>&1
ls -la gpurun_out/src_*
