"""Generates tests/golden/*.json from the VERBATIM reference engine
(oracle/_ref, compiled from /root/reference/proj by oracle/Makefile).

Run in the build container (needs oracle/_ref):  python tests/golden/make_golden.py

Fixtures (all inputs produced by the reference's own seeded generators):
  ref_kats.json      reference known answers: single event (test_likelihood.cpp:42-56),
                     5-event fixture (:84-104), theta=0 instance (:58-82),
                     underflow instance (:156-175)
  ref_random.json    the 32 random instances of test_likelihood.cpp:106-121
                     (Rng(2024) params, cloud seeds 1000+k, N in {2,3,10,100})
                     with the reference loglik (serial and threads4+simd4)
  ref_c1.json        C1: generateBenchmarkCloud(1000,{0,4,0,4,60},Rng(1000)) at
                     Theta=(0.6,0.9,3,0.5,1.1,0.35): events, loglik, per-event terms
  ref_sim.json       generator checksums (cloud + cluster C2) for the sim restatement
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_glue as og  # noqa: E402


def mt_uniform_params(seed, count):
    """Reproduce test_likelihood.cpp:24-32 randomParams draws from Rng(seed):
    uniform(lo,hi) = lo + (hi-lo)*u with u=(mt19937_64()>>11)*2^-53."""
    gen = MT19937_64(seed)
    out = []
    for _ in range(count):
        u = lambda lo, hi: lo + (hi - lo) * ((gen.next() >> 11) * 2.0 ** -53)
        out.append([u(0.3, 2.0), u(0.5, 2.0), u(2.0, 20.0), u(0.05, 0.8), u(0.3, 3.0),
                    u(0.1, 1.0)])
    return out


class MT19937_64:
    """std::mt19937_64 (bit-specified by the C++ standard)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def next(self):
        if self.idx >= 312:
            for i in range(312):
                x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def main():
    assert og.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    kats = {}
    x, y, t = [0.0], [0.0], [1.0]
    ll, ok, _ = og.ref_loglik(x, y, t, 1.0, [1, 1, 1, 1, 1, 1])
    kats["single_event"] = dict(x=x, y=y, t=t, T=1.0, params=[1, 1, 1, 1, 1, 1], loglik=ll,
                                valid=ok, frozen=-3.0981603456825612)
    x5 = [0.1, 0.9, -0.4, 0.2, 1.1]
    y5 = [-0.2, 0.3, 0.5, 0.9, -0.8]
    t5 = [0.4, 1.1, 1.9, 3.0, 4.2]
    p5 = [0.6, 0.9, 3.0, 0.5, 1.1, 0.35]
    ll, ok, pe = og.ref_loglik(x5, y5, t5, 5.0, p5, per_event=True)
    kats["five_event"] = dict(x=x5, y=y5, t=t5, T=5.0, params=p5, loglik=ll, valid=ok,
                              per_event=pe.tolist())
    # theta = 0 (test_likelihood.cpp:58-82 uses randomEvents(40,11), randomParams(Rng(12)))
    cx, cy, ct, cwe = og.ref_sim_cloud(40, [0, 4, 0, 4, 60], 11)
    p0 = mt_uniform_params(12, 1)[0]
    p0[3] = 0.0
    ll, ok, _ = og.ref_loglik(cx, cy, ct, cwe, p0)
    kats["theta_zero"] = dict(x=cx.tolist(), y=cy.tolist(), t=ct.tolist(), T=cwe, params=p0,
                              loglik=ll, valid=ok)
    pu = [5e-324, 1e120, 1e120, 0.0, 1.0, 1.0]
    ll, ok, _ = og.ref_loglik([0.0, 1.0], [0.0, 0.0], [0.0, 1.0], 1.0, pu)
    kats["underflow"] = dict(x=[0.0, 1.0], y=[0.0, 0.0], t=[0.0, 1.0], T=1.0, params=pu,
                             loglik=None if not np.isfinite(ll) else ll, valid=ok)
    json.dump(kats, open(os.path.join(HERE, "ref_kats.json"), "w"), indent=1)

    rnd = []
    params = mt_uniform_params(2024, 32)
    inst = 0
    for n in (2, 3, 10, 100):
        for _ in range(8):
            x, y, t, we = og.ref_sim_cloud(n, [0, 4, 0, 4, 60], 1000 + inst)
            p = params[inst]
            ll_s, ok_s, _ = og.ref_loglik(x, y, t, we, p)
            ll_v, ok_v, _ = og.ref_loglik(x, y, t, we, p, threads=4, lanes=4)
            rnd.append(dict(n=n, seed=1000 + inst, x=x.tolist(), y=y.tolist(), t=t.tolist(),
                            T=we, params=p, loglik_serial=ll_s, loglik_t4s4=ll_v,
                            valid=ok_s and ok_v))
            inst += 1
    json.dump(rnd, open(os.path.join(HERE, "ref_random.json"), "w"))

    x, y, t, we = og.ref_sim_cloud(1000, [0, 4, 0, 4, 60], 1000)
    p = [0.6, 0.9, 3.0, 0.5, 1.1, 0.35]
    ll, ok, pe = og.ref_loglik(x, y, t, we, p, per_event=True)
    ll8, _, _ = og.ref_loglik(x, y, t, we, p, threads=8, lanes=8)
    json.dump(dict(seed=1000, window=[0, 4, 0, 4, 60], T=we, params=p, loglik_serial=ll,
                   loglik_t8s8=ll8, valid=ok, x=x.tolist(), y=y.tolist(), t=t.tolist(),
                   per_event=pe.tolist()),
              open(os.path.join(HERE, "ref_c1.json"), "w"))

    sim = {}
    for n, w, seed in [(1000, [0, 4, 0, 4, 60], 1000), (85000, [0, 15, 0, 15, 4750], 85000)]:
        x, y, t, we = og.ref_sim_cloud(n, w, seed)
        sim[f"cloud_{n}_{seed}"] = dict(n=n, window=w, seed=seed, sha_x=sha(x), sha_y=sha(y),
                                        sha_t=sha(t))
    x, y, t, par = og.ref_sim_cluster([1, 1.6, 14, 0.344, 1440, 0.0695], [0, 15, 0, 15, 4750],
                                      0.053217, 2005)
    sim["cluster_c2"] = dict(params=[1, 1.6, 14, 0.344, 1440, 0.0695], window=[0, 15, 0, 15, 4750],
                             rate=0.053217, seed=2005, n=int(t.size), sha_x=sha(x), sha_y=sha(y),
                             sha_t=sha(t), sha_parent=hashlib.sha256(par.tobytes()).hexdigest(),
                             t_85000=float(t[84999]))
    json.dump(sim, open(os.path.join(HERE, "ref_sim.json"), "w"), indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
