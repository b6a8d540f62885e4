python -m pytest tests -m gpu -x -q -k "ssim or mapping_objective" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
