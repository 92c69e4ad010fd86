"""Host (LAPACK) vs device (cuSOLVER, acpf_zbus_reduce) Z-Bus network reduction time."""
import sys, time
sys.path.insert(0, '.')
import paper_2605_14103_b200 as pf
from paper_2605_14103_b200.fixtures import load_distribution

for name in sys.argv[1:] or ['ieee13', 'ieee123', 'eulv']:
    net = load_distribution(name)
    pf.build_zbus_model(net, device=0)  # warm-up (context, cuSOLVER handle)
    for dev in (None, 0):
        t0 = time.perf_counter()
        m = pf.build_zbus_model(net, device=dev)
        t = time.perf_counter() - t0
        print(f"{name}: n={m.n} |l|={m.load_cols.size} reduce on {'host' if dev is None else 'GPU'}: {t*1e3:.1f} ms",
              flush=True)
