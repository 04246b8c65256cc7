#!/bin/bash
set -u
python -c "import __graft_entry__ as E; E.build()" > /dev/null 2>&1
OPTS='"" dsmem=0 dsmem=0,tlanes=512 lanes=384 dsmem=0,lanes=512' WL="tf96" bash tools/jit_sweep.sh
