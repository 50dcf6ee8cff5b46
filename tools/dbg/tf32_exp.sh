#!/bin/bash
# S_cq pipeline experiments: kernel time with parts of the pipeline disabled
for d in ${@:-0 7}; do
  echo "dbg=$d"; PLAID_TF32_DBG=$((d+16)) python tools/tf32_timeline.py 2>&1 | grep -E "scores_ms|span|Error|error"
done
