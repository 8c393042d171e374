# one ncu --set full capture per hot kernel (single GPU, one process at a time) + the bench launch list.
# Reports are summarised on the box (raw metrics -> JSON, SASS hot spots -> text) and the .ncu-rep
# files are dropped unless KEEP_REP=1 (gpurun copies back at most 64 MiB).
set -x
NCU=/usr/local/cuda/bin/ncu
export PATH=/usr/local/cuda/bin:$PATH
TAG=${TAG:-r1v4}
mkdir -p gpurun_out
cap() {  # name workload kernel-regex
  timeout 600 $NCU --set full --clock-control none --import-source on -k "regex:$3" -s 2 -c 1 \
     -o gpurun_out/${TAG}_$1 -f python tools/prof.py $2 4 > gpurun_out/${TAG}_$1.log 2>&1
  python tools/ncu_export.py gpurun_out/${TAG}_$1_summary.json gpurun_out/${TAG}_$1.ncu-rep >> gpurun_out/${TAG}_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/${TAG}_$1.ncu-rep > gpurun_out/${TAG}_$1_metrics.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${TAG}_$1.ncu-rep "$3" > gpurun_out/${TAG}_$1_sass_hot.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/${TAG}_$1.ncu-rep
}
CAPS=${CAPS:-"czt64:czt64:k_czt_sf czt32:czt32:k_czt_sf cube32:cube32:k_fft_r2c zoom64:zoom64:k_zoom_pfir zoom32:zoom32:k_zoom_pfir"}
for spec in $CAPS; do
  IFS=: read -r a b c <<< "$spec"
  cap "$a" "$b" "$c"
done
if [ -z "$NOLAUNCH" ]; then
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1
fi
du -sh gpurun_out; ls -la gpurun_out
