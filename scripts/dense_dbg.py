import sys
sys.path.insert(0, '.')
import paper_1408_3877_b200 as ld
dim = int(sys.argv[1]); ps = [int(x) for x in sys.argv[2].split(',')]
for p in ps:
    s = ld.LdgSystem.square(dim, p, ld.BASELINE_SPEC)
    s.initial_state()
    st = s.euler_steps(0.05, 2)
    print(p, st['iterations'], st['residual'], flush=True)
    s.close()
