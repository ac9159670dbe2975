import sys, time
sys.path.insert(0, '.')
import paper_1306_6291_b200 as sd
m = sd.SymMat3(1.0, 2.0, 3.0, 0.1, 0.2, 0.3)
m2 = sd.SymMat2(1.0, 2.0, 0.3)
for f, arg, name in ((sd.diagonalize3, m, "diagonalize3"), (sd.diagonalize2, m2, "diagonalize2")):
    for _ in range(20): f(arg)
    t = time.perf_counter()
    for _ in range(500): f(arg)
    print(name, (time.perf_counter() - t) / 500 * 1e6, "us/call")
