# quick A/B sweeps (ms per step)
ms() { python bench.py "$@" --steps 5 --warmup 3 --no-cpu --single 2>/dev/null | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("%.4f"%d["ms_per_step"], [(p["m"],p["n"],p["block"]) for p in d["details"]["plan"]], d["details"]["kernel"])'; }
for m in 768,768,1024 768,768,512 768,768,768 384,768,1024 768,384,1024 768,768,384; do echo "c5 $m $(ms --config c5 --m $m)"; done
echo "c5 planner $(ms --config c5)"
