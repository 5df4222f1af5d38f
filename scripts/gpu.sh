#!/bin/bash
# build the sm_100a library locally (it travels with the snapshot), then run $1 on a B200
set -e
cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; exit 1; }
exec /usr/local/graft/bin/gpurun --timeout "${2:-1800}" -- bash "$1"
