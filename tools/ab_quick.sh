# quick correctness + A/B: sampler GPU tests, then ab_env.sh over $VARIANTS
timeout 900 python -m pytest tests/test_sampler_gpu.py tests/test_trainer_gpu.py -x -q --timeout 600 2>&1 | tail -3
bash tools/ab_env.sh
