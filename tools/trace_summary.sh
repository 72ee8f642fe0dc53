#!/bin/bash
# one line per probe_trace log: seconds, kkt, outer iterations, per-class device ms
for f in "$@"; do tail -n 1 $f | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['prof']; print('$f'.split('/')[-1], round(d['seconds'],3), '%.2e'%d['kkt'], d['outer_iters'], {k:round(v['ms']) for k,v in p.items() if v['ms']>1})"; done
