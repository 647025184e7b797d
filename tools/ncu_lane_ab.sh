# instruction counts / durations of the lane kernels (sequential mode) for the library variants in $LIBS
for v in "" ${LIBS}; do
  tag=$(echo "base$v" | tr ' =/.' '____')
  A3G_LIB=$v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.avg --clock-control none -k regex:k_stream_lane -c 4 --csv python bench.py --steps 2 --warmup 2 --pipeline 0 --no-cpu-baseline 2>/dev/null | grep k_stream_lane | awk -F'","' -v t="$tag" '{print t, $5, $(NF-2), $NF}' | tr -d '"'
done
bash tools/ab_env.sh
