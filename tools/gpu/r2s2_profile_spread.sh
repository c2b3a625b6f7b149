# ncu of the spread small round at C1 (eager rounds: a graph replay is not profiled)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1 SPREAD_NO_GRAPH=1 MARSIT_SPREAD_COOP=0  # ncu fails cooperative cluster launches
O=gpurun_out/prof2
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:round_spread_kernel" -s 30 -c 1 \
    -o $O/spread -f python tools/spread_probe.py > $O/ncu_spread.log 2>&1; echo spread_rc=$?
python tools/ncu_summary.py $O/spread.ncu-rep > $O/ncu_spread_summary.txt 2>&1
ncu -i $O/spread.ncu-rep --page source --csv --print-source sass > $O/spread_sass.csv 2>/dev/null; echo sass_rc=$?
grep -c "UTCBAR\|STTM\|LDTM\|UTMALLOC" $O/spread_sass.csv
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/spread_launches.csv python tools/spread_probe.py > /dev/null 2>&1; echo spread_launches_rc=$?
mv $O/spread.ncu-rep $O/../spread_c1.ncu-rep
ls -la $O
