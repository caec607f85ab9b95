RHG_TIMELINE=1 timeout 100 python -c "
import sys; sys.path.insert(0,'.')
import paper_1710_07565_b200 as rhg
p = rhg.ModelParams.from_avg_degree(1 << 24, rhg.alpha_from_gamma(2.2), 64.0, 7, 64)
for _ in range(3): rhg.generate_stats(p, rhg.GenOptions(rank=${R:-7}, world=${W:-8}))
" 2>&1 | grep TIMELINE | tail -1
