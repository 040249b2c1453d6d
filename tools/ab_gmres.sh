for r in 1 2; do
for L in paper_1104_3349_b200/libmscg_a.so paper_1104_3349_b200/libmscg.so; do
  MSCG_LIB=$PWD/$L timeout 300 python bench.py --config cfg2 --mode gmres > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$L', d['iterations'], 'solve_s %.3f'%d['solve_s'])"
done; done
