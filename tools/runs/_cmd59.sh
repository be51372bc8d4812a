python -m paper_2604_16395_b200.build --force > /dev/null
echo "== gpu tests"; timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
bash tools/round_evidence.sh r01g
