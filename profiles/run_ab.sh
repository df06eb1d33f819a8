OUT=gpurun_out
echo "== octet register k_fine"; timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
bash profiles/run_quick.sh 2>&1 | grep -v passed | tail -6
cp paper_2603_08453_b200/variants/liblychee_b200_cp.so paper_2603_08453_b200/liblychee_b200.so
echo "== cp.async k_fine"; timeout 600 python -m pytest tests -x -q -m gpu -k "parity" 2>&1 | tail -1
bash profiles/run_quick.sh 2>&1 | grep -v passed | tail -6
