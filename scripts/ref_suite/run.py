"""Stage the reference tests (baseline/_ref/ref_tests) with the drop-in conftest and run them."""
import os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tests = os.path.join(ROOT, "baseline", "_ref", "ref_tests")
shutil.copy(os.path.join(ROOT, "scripts", "ref_suite", "conftest.py"), os.path.join(tests, "conftest.py"))
env = dict(os.environ, VLMP_REPO=ROOT, PYTHONDONTWRITEBYTECODE="1")
sys.exit(subprocess.call([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-rf", tests] + sys.argv[1:], env=env, cwd=tests))
