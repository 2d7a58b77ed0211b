timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "FAILED|Error|error|assert" | head -20
