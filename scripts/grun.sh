#!/bin/bash
# build here, then run "$2" on the GPU box; log under gpurun_out/$1.log (development helper)
cd /root/repo || exit 1
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { grep -i error /tmp/build.log | head; exit 1; }
/usr/local/graft/bin/gpurun --timeout ${GT:-1200} -- "$2" > gpurun_out/$1.log 2>&1
tail -1 gpurun_out/$1.log
