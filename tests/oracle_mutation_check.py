"""Mutation check for the oracle pins (run manually: python tests/oracle_mutation_check.py).
Each mutation is a plausible slip in the scheme; every one must fail >=1 pin.
Mutations 11-16 are slips in the order-2 (MUSCL-Hancock + FORCE) path.
Last run: all 16 mutations caught."""
import subprocess, sys, shutil
muts = [
 ("(REAL)0.5 * (dx / dt) * (R[c] - L[c])", "(REAL)0.25 * (dx / dt) * (R[c] - L[c])", "LF diffusion coeff"),
 ("(REAL)0.5 * (dt / dx) * (FR[c] - FL[c])", "(REAL)0.5 * (dx / dt) * (FR[c] - FL[c])", "RI dt/dx swapped"),
 ("F[D + 1] = (E + p) * ud;", "F[D + 1] = E * ud;", "energy flux drops p"),
 ("if (k == d) F[1 + k] = F[1 + k] + p;", "if (k == d) F[1 + k] = F[1 + k];", "momentum flux drops p"),
 ("REAL p = gm1 * (E - ke);", "REAL p = gm1 * (E - (REAL)2 * ke);", "EOS kinetic factor"),
 ("if (flip) dst[1 + d] = -dst[1 + d];", "", "reflective no flip"),
 ("Uo[c] = Ui[c] - (dt / dx) *", "Uo[c] = Ui[c] + (dt / dx) *", "update sign"),
 ("for (int c = 0; c < C; ++c) Fout[c] = (REAL)0.5 * (Flf[c] + Fri[c]);", "for (int c = 0; c < C; ++c) Fout[c] = Flf[c];", "FORCE -> LF only"),
 ("REAL ud = U[1 + d] * inv;", "REAL ud = U[1] * inv;", "velocity index fixed to x"),
 ("src = ((t % N) + N) % N;", "src = ((t % N) + N + 1) % N;", "periodic off by one"),
 ("if (a > 0 && b > 0) return a < b ? a : b;", "if (a > 0 && b > 0) return a > b ? a : b;", "o2: limiter picks larger"),
 ("  return 0;\n}\n\n/* MUSCL", "  return (REAL)0.5 * (a + b);\n}\n\n/* MUSCL", "o2: no limiting at extrema"),
 ("UL[c] = U0[c] - (REAL)0.5 * delta;", "UL[c] = U0[c] - delta;", "o2: full slope on left"),
 ("UbL[c] = UL[c] + (REAL)0.5 * (dt / dx) * (FL[c] - FR[c]);", "UbL[c] = UL[c] - (REAL)0.5 * (dt / dx) * (FL[c] - FR[c]);", "o2: half-step sign (L)"),
 ("UbR[c] = UR[c] + (REAL)0.5 * (dt / dx) * (FL[c] - FR[c]);", "UbR[c] = UR[c];", "o2: no half-step (R)"),
 ("UbR + C * f, UbL + C * (f + 1)", "UbL + C * f, UbR + C * (f + 1)", "o2: face takes wrong sides"),
]
shutil.copy('oracle/oracle_scheme.inc', '/tmp/orig.inc'); orig = open('/tmp/orig.inc').read()
for a, b, name in muts:
    assert a in orig, name
    open('oracle/oracle_scheme.inc','w').write(orig.replace(a, b))
    r = subprocess.run([sys.executable, '-m', 'pytest', 'tests/test_oracle_pins.py', '-q', '-p', 'no:cacheprovider'], capture_output=True, text=True)
    last = r.stdout.strip().splitlines()[-1]
    print(f"{name:32s} -> {last}")
open('oracle/oracle_scheme.inc','w').write(orig)
