python -m pytest tests -m gpu -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
python -c "import __graft_entry__ as g; g.smoke()"
