#!/bin/bash
# gpurun from the repo root (results merge into /root/repo/gpurun_out)
cd /root/repo && exec /usr/local/graft/bin/gpurun "$@"
