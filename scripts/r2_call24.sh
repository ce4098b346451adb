#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_graph.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider 2>&1 | tail -15
IG_SEQ_SEEDS=24 timeout 1800 python -m pytest tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider 2>&1 | tail -3
