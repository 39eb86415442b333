start=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 2>&1 | tail -15
echo "wall=$(( $(date +%s) - start ))s"
