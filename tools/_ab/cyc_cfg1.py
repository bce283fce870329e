import runpy, sys
sys.path.insert(0, ".")
import paper_1604_02614_b200.fdjac as F
orig = F.FdJacobianOperator.__init__
def init(self, *a, **k):
    orig(self, *a, **k)
    self._matvec = self._apply     # the old reference cycle
F.FdJacobianOperator.__init__ = init
sys.argv = ["run_configs.py", "--config", "1"]
runpy.run_path("tools/run_configs.py", run_name="__main__")
