#!/bin/bash
# launch lists (shares) of the generalized reorder (C5 construction, n=8000)
# and of the Hessenberg reduction (n=4000)
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python tools/c5_small.py 8000 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c5.csv "C5 construction n=8000 (tools/c5_small.py)" > $O/r03_launches_c5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_hess.csv python tools/hess_time.py 4000 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_hess.csv "Hessenberg n=4000 (tools/hess_time.py, 2 reps)" > $O/r03_launches_hess.txt 2>&1
cat $O/r03_launches_c5.txt $O/r03_launches_hess.txt
