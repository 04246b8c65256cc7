#!/bin/bash
set -u
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
OPTS='"" lanes=384 lanes=512 lanes=768' WL="ws30 rn50f iv3f tf96 ws_stack_10x100" bash tools/jit_sweep.sh
