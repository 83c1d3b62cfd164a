"""Numerics of the d=2 LSE sum-kernel tune variants (SKNR_SUM_VARIANT, tile_kernels.cu
tune_variant): each variant runs in its own process at BASELINE C4 shape; both transforms
of a random f and 20 SK iterations are compared with the default kernel, and the column
transform of a 4096-point C4-shaped problem with the oracle.
  python tools/variant_check.py 50 52 ...      (prints one JSON line per variant)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np

    import paper_2506_14780_b200 as sk
    from paper_2506_14780_b200 import generators as G

    c = G.config("C4")
    p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon)
    f = 0.02 * np.random.default_rng(4).standard_normal(c.n)
    g = sk.ctransform_of_f(p, f)
    f2 = sk.ctransform_of_g(p, g)
    r = sk.solve(p, tol=1e-300, max_iter=20, trace=False)
    out = {"g": g, "f2": f2, "sk_f": r.f}
    small = G.config("C4", n=4096, m=4096)
    ps = sk.PointProblem(small.x, small.y, small.alpha, small.beta, small.epsilon)
    fs = 0.02 * np.random.default_rng(5).standard_normal(small.n)
    out["small_g"] = sk.ctransform_of_f(ps, fs)
    if os.environ.get("SKNR_SUM_VARIANT") is None:
        import oracle_ref as O

        op = O.Instance(small.alpha, small.beta, small.epsilon, x=small.x, y=small.y)
        out["small_oracle"] = O.ctransform_of_f(op, fs)
    np.savez(sys.argv[2], **out)


def main():
    import numpy as np

    tmp = os.path.join(ROOT, "gpurun_out", "variant_check")
    os.makedirs(tmp, exist_ok=True)
    base = os.path.join(tmp, "base.npz")
    env = dict(os.environ)
    env.pop("SKNR_SUM_VARIANT", None)
    subprocess.run([sys.executable, __file__, "--child", base], env=env, check=True)
    b = np.load(base)

    def rel(a, c):
        return float(np.max(np.abs(a - c)) / np.max(np.abs(c)))

    print(json.dumps({"variant": "default", "small_vs_oracle": rel(b["small_g"], b["small_oracle"])}), flush=True)
    for v in sys.argv[1:]:
        path = os.path.join(tmp, f"v{v}.npz")
        env["SKNR_SUM_VARIANT"] = v
        rc = subprocess.run([sys.executable, __file__, "--child", path], env=env).returncode
        if rc != 0:
            print(json.dumps({"variant": int(v), "error": rc}), flush=True)
            continue
        d = np.load(path)
        print(json.dumps({"variant": int(v), "g_vs_default": rel(d["g"], b["g"]), "f2_vs_default": rel(d["f2"], b["f2"]),
                          "sk20_f_vs_default": rel(d["sk_f"], b["sk_f"]),
                          "small_vs_oracle": rel(d["small_g"], b["small_oracle"])}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        main()
