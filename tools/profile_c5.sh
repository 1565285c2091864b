mkdir -p gpurun_out
bash tools/profile_all.sh c5 c4
for f in c5 c4; do python -c "
import json
for r in json.load(open('gpurun_out/launches_${f}_summary.json'))[:6]: print('$f %6d %10.1f us %5.3f %8.2f avg  %s'%(r['launches'],r['total_us'],r['share'],r['avg_us'],r['kernel'][:100]))
"; done
