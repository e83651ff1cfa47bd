make -s -C oracle >/dev/null 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x -p dropin_plugin 2>&1 | tail -6
