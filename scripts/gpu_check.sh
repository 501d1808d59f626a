nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
python -c "import paper_2106_04487_b200 as f; print(f.lib.fkt_version())"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1" 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -40
