SKG_ZOOM_NO_FUSE=1 python tools/zoom_time.py 30
M=gpu__time_duration.sum
SKG_ZOOM_NO_FUSE=1 ncu --metrics $M --clock-control none -k regex:zoom --csv --log-file gpurun_out/r12_zoom_nofuse.csv python tools/zoom_time.py 2 > /dev/null 2>&1
grep -v "^==" gpurun_out/r12_zoom_nofuse.csv | awk -F'","' '{print $5, $(NF)}' | tail -16
