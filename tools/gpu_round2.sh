timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "passed|failed|PASSED.*boundary" | tail -4
