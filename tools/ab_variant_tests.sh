# sampler parity under each variant library, then the A/B
for v in ${LIBS}; do
  A3G_LIB=$v timeout 900 python -m pytest tests/test_sampler_gpu.py -x -q --timeout 600 2>&1 | tail -1 | sed "s|^|$v: |"
done
bash tools/ab_env.sh
