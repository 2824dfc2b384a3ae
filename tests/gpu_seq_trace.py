import sys; sys.path.insert(0,'.')
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
for name in sys.argv[1:]:
    c=CONFIGS[name]; r=S.hqdwh(make_input(name), c["nmin"], c["eps"])
    t=S.micro_kernel(5,0,0)
    f=1965e3
    print(name, "LU %.1f ms, Hager %.1f ms, Givens %.1f ms" % ((t[1]-t[0])/f, (t[2]-t[1])/f, (t[4]-t[3])/f), "setup", round(r.info["ms_setup"],1), "first", round(r.info["ms_first"],1))
