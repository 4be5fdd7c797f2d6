bash tools/gpu/ctl.sh 2>&1 | grep -A10 "^warp"
python -m pytest tests -m gpu -x -q -k "not full" 2>&1 | tail -3
python tools/prof_step.py --trace 2>&1 | tail -10
