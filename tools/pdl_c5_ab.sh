for r in 1 2 3; do for v in on off; do
 if [ $v = off ]; then export TOMESH_NO_PDL=1; else unset TOMESH_NO_PDL; fi
 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c5 pdl=$v', round(d['value'],1), round(r['avg_launch_ms']*1000,2), round(r['frac'],4))"
done; done
