import sys; sys.path.insert(0, ".")
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
c = CONFIGS["banded"]; r = S.hqdwh(make_input("banded"), c["nmin"], c["eps"]); print(r.l0)
