set -x
nproc; cat /proc/meminfo | head -3; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
