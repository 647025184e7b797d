#!/bin/bash
# build here, then (only if the build succeeded) run tools/gpu_quick.sh on the box
cd /root/repo
python -c "from paper_2511_07421_b200 import build as b; b.build()" > /tmp/build.log 2>&1 || { echo "BUILD FAILED"; grep -E "error" /tmp/build.log | head; exit 1; }
timeout 2400 /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1500} -- "CONFIGS=\"${CONFIGS:-c2}\" BENCH_ARGS=\"${BENCH_ARGS:-}\" PYTEST_ARGS=\"${PYTEST_ARGS:-}\" bash tools/gpu_quick.sh" 2>&1 | tail -8 | cut -c1-260
