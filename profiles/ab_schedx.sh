for w in ${WLS:-cfg1 cfg0 cfg4_L8 cfg4_L32 fa_i8_4.5 fa_i16_4.5}; do
for lib in /root/repo/paper_1710_08314_b200/libpolar_base.so ""; do
PLB_LIB=$lib python bench.py --workload $w --extra none --steps 10 --no-cpu --e2e-steps 1 2>/dev/null | python -c "
import sys,json
for ln in sys.stdin:
    if ln.startswith('{'):
        d=json.loads(ln); print('${lib:-NEW}'.split('/')[-1], d['config']['workload'], round(d['value'],3))
"
done; done
