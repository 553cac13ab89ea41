"""Mutation check of the oracle pins: apply plausible mistakes to a copy of
oracle/hsgn_oracle.c and confirm that `pytest tests/test_oracle_pins.py` fails
for every one of them.  Dev tool; not part of the product or of the test suite.

    python tools/mutation_check.py
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "hsgn_oracle.c")).read()

MUTANTS = {
    "R2 reading of A1 (mean delta with 1/(2dx^2))":
        ("const double lt2 = lam * tau * tau / (2.0 * dx * dx);",
         "const double lt2 = lam * tau * tau / (4.0 * dx * dx);"),
    "sign of tau*W^dagger in H^dagger":
        ("- 1.5 * tau * qE * Dxb[i] + tau * Wd_;", "- 1.5 * tau * qE * Dxb[i] - tau * Wd_;"),
    "beta2 missing factor 2":
        ("double beta2 = 2.0 * lambda", "double beta2 = 1.0 * lambda"),
    "transposed hbar neighbours in qbar":
        ("be[i + 1] * (hr - hl)", "be[i + 1] * (hl - hr)"),
    "Rusanov speed min instead of max":
        ("double a = fabs(um) > fabs(up_) ? fabs(um) : fabs(up_);",
         "double a = fabs(um) < fabs(up_) ? fabs(um) : fabs(up_);"),
    "Rusanov dissipation sign":
        ("- 0.5 * a * (vp[1] - vm[1]);", "+ 0.5 * a * (vp[1] - vm[1]);"),
    "H flux uses q instead of H":
        ("out[1] = 0.5 * (vm[2] * um + vp[2] * up_)", "out[1] = 0.5 * (vm[1] * um + vp[1] * up_)"),
    "p-tilde sign in momentum bathymetric source":
        ("- 1.5 * tau * ptil * Dxb[i];", "+ 1.5 * tau * ptil * Dxb[i];"),
    "hydrostatic back-substitution term sign":
        ("- tau * g * X(eh, i) * Dxb[i];", "+ tau * g * X(eh, i) * Dxb[i];"),
    "MUSCL slope not halved":
        ("double s0 = (X(ev[k], f + 1) - X(ev[k], f - 1)) / 2.0;",
         "double s0 = (X(ev[k], f + 1) - X(ev[k], f - 1)) / 1.0;"),
    "dropped lambda*tau source in W^dagger":
        ("+ lam * tau;\n", ";\n"),
    "Hbar uses beta1 at E instead of hbar":
        ("double Hn = Hd[i + 1] / (1.0 + lam * tau * tau / (hn * hn));",
         "double Hn = Hd[i + 1] / (1.0 + lam * tau * tau / (X(eh, i) * X(eh, i)));"),
    "a2 = c2 + lambda eta alpha":
        ("double a2 = c2 - lambda * eta * alpha;", "double a2 = c2 + lambda * eta * alpha;"),
    "wE/wR swapped":
        ("*wE = T->aE[1][0] / T->aI[0][0];\n    *wR = T->aI[1][0] / T->aI[0][0];",
         "*wR = T->aE[1][0] / T->aI[0][0];\n    *wE = T->aI[1][0] / T->aI[0][0];"),
    "wall q parity even":
        ("const double qpar = -1.0;", "const double qpar = 1.0;"),
    "delta uses beta1^2":
        ("double delta = alpha / beta1;", "double delta = alpha / (beta1 * beta1);"),
    "bathymetry source in H^dagger sign":
        ("- 1.5 * tau * qE * Dxb[i] + tau * Wd_;", "+ 1.5 * tau * qE * Dxb[i] + tau * Wd_;"),
    "hydrostatic zeta term dropped":
        ("hd = hd + t2 * (Gr * dbr - Gl * dbl);", "hd = hd + 0.0 * t2 * (Gr * dbr - Gl * dbl);"),
    "nu_max from P:628 literal":
        ("return sqrt(g * h + (lambda / 3.0) * eta_over_h * eta_over_h);",
         "return sqrt(g * h + (lambda / 3.0) * (eta_over_h - 1.0));"),
}
# A25 (well-balanced face form) mutants: checked against tests/test_oracle_wb.py
WB_MUTANTS = {
    "A25 dhat sign of (2 sigma - 1)":
        ("return -(2.0 * sig - 1.0) / (3.0 * ht) * bt;", "return -(2.0 * sig + 1.0) / (3.0 * ht) * bt;"),
    "A25 dhat one-sided 1/beta1":
        ("double sig = 0.5 * (s0 + s1), ht = 0.5 * (h0 + h1), bt = 0.5 * (b0 + b1);",
         "double sig = 0.5 * (s0 + s1), ht = 0.5 * (h0 + h1), bt = b0;"),
    "A25 mu without the factor 2":
        ("ml = 2.0 * lt2 * wb_delta(eh, eH, i - 1, lam, tau, G);",
         "ml = 1.0 * lt2 * wb_delta(eh, eH, i - 1, lam, tau, G);"),
    "A25 face hydrostatic term dropped (right face)":
        ("+ 0.5 * g * (X(eh, i) + X(eh, i + 1)) * (X(eb, i + 1) - X(eb, i));",
         "+ 0.0 * g * (X(eh, i) + X(eh, i + 1)) * (X(eb, i + 1) - X(eb, i));"),
    "A25 qbar face fluxes subtracted with the wrong sign":
        ("qn = qd[i + 1] - (tau / (2.0 * dx)) * (Phr + Phl);", "qn = qd[i + 1] - (tau / (2.0 * dx)) * (Phr - Phl);"),
}

# explicit hSGN scheme (A22) mutants: tests/test_oracle_explicit.py
EX_MUTANTS = {
    "explicit: centred mass flux sign":
        ("L[0][i] = -Dxq;", "L[0][i] = +Dxq;"),
    "explicit: pressure term lam alpha DxH dropped":
        ("- a2 * Dxh - lam * alpha * DxH;", "- a2 * Dxh;"),
    "explicit: W relaxation source sign":
        ("- lam * (H / (h * h) - 1.0);", "+ lam * (H / (h * h) - 1.0);"),
    "explicit: Heun weight 1/2 -> 1":
        ("U[k][i] = 0.5 * Un[k][i] + 0.5 * (U1[k][i] + dt * Lb[k][i]);",
         "U[k][i] = 0.0 * Un[k][i] + 1.0 * (U1[k][i] + dt * Lb[k][i]);"),
}
# classical SGN scheme (A23) mutants: tests/test_oracle_sgn.py
SGN_MUTANTS = {
    "SGN: h* with g h instead of g h^3 (the literal P:591)":
        ("* (g * hp3 * (XS(eh, i + 2) - 2.0 * hp + XS(eh, i))", "* (g * hp * (XS(eh, i + 2) - 2.0 * hp + XS(eh, i))"),
    "SGN: phi system off-diagonal h^3/3 -> h^3":
        ("double cl = hl * hl * hl / (3.0 * dx * dx), cr = hr * hr * hr / (3.0 * dx * dx);",
         "double cl = hl * hl * hl / (1.0 * dx * dx), cr = hr * hr * hr / (1.0 * dx * dx);"),
    "SGN: source h phi sign":
        ("Lq[i] = -(Fq[i + 1] - Fq[i]) / dx + XS(eh, i) * phi[i];",
         "Lq[i] = -(Fq[i + 1] - Fq[i]) / dx - XS(eh, i) * phi[i];"),
    "SGN: Rusanov speed without sqrt(g h)":
        ("double am = fabs(um) + sqrt(g * vm[0]), ap = fabs(up_) + sqrt(g * vp[0]);",
         "double am = fabs(um), ap = fabs(up_);"),
}
# bathymetric SGN closure (A26) mutants: tests/test_oracle_sgnb.py
SGNB_MUTANTS = {
    "SGNb: hydrostatic source g h b_x dropped (the literal P:566)":
        ("if (P->b) Lq[i] -= g * XS(eh, i)", "if (0) Lq[i] -= g * XS(eh, i)"),
    "SGNb: kappa 3/4 h b_x^2 term sign":
        ("+ 0.75 * XS(eh, i) * bx * bx;", "- 0.75 * XS(eh, i) * bx * bx;"),
    "SGNb: rho hydrostatic part sign":
        ("rho[s2] = -(hj * hj * bx / 2.0) * g * zx", "rho[s2] = +(hj * hj * bx / 2.0) * g * zx"),
    "SGNb: Q without the 3 g b_x zeta_x / 4 term":
        ("- (3.0 * g * bx / 4.0) * zx + h0 * ux * ux", "+ 0.0 * zx + h0 * ux * ux"),
    "SGNb: g-term on h instead of zeta":
        ("* (g * hp3 * (XZ(i + 2) - 2.0 * XZ(i + 1) + XZ(i))", "* (g * hp3 * (XS(eh, i + 2) - 2.0 * hp + XS(eh, i))"),
}

# operator-split extras and the Picard pass: tests/test_oracle_pins_ops.py
OPS_MUTANTS = {
    "A19 filter sigma/16 -> sigma/8":
        ("U[k][i] = ext[i + 2] - (P->filter_sigma / 16.0) * d4;",
         "U[k][i] = ext[i + 2] - (P->filter_sigma / 8.0) * d4;"),
    "Picard pass beta2 factor 2 -> 1":
        ("double beta2 = 2.0 * lam * tau * tau / (beta1 * beta1 * hb * hb * hb);",
         "double beta2 = 1.0 * lam * tau * tau / (beta1 * beta1 * hb * hb * hb);"),
    "Picard pass delta = alpha (not alpha/beta1)":
        ("de[i + 1] = alE[i] / beta1;", "de[i + 1] = alE[i];"),
    "sponge ramp r^2 -> r":
        ("double r = (x - P->sp_x0) / (x_max - P->sp_x0);\n            s = P->sp_rate * r * r;",
         "double r = (x - P->sp_x0) / (x_max - P->sp_x0);\n            s = P->sp_rate * r;"),
    "A19 filter stencil not conservative (6 -> 5)":
        ("6.0 * ext[i + 2]", "5.0 * ext[i + 2]"),
    "A19 filter q ghost parity even at walls":
        ("double par = (k == 1) ? -1.0 : 1.0;", "double par = 1.0;"),
    "wavemaker target velocity halved":
        ("double u = P->cp * eta / P->level;", "double u = 0.5 * P->cp * eta / P->level;"),
}

ok = True
for name, (a, b), tf in [(k, v, "test_oracle_pins.py") for k, v in MUTANTS.items()] + \
                        [(k, v, "test_oracle_wb.py") for k, v in WB_MUTANTS.items()] + \
                        [(k, v, "test_oracle_explicit.py") for k, v in EX_MUTANTS.items()] + \
                        [(k, v, "test_oracle_sgn.py") for k, v in SGN_MUTANTS.items()] + \
                        [(k, v, "test_oracle_sgnb.py") for k, v in SGNB_MUTANTS.items()] + \
                        [(k, v, "test_oracle_pins_ops.py") for k, v in OPS_MUTANTS.items()]:
    assert SRC.count(a) >= 1, name
    if len(sys.argv) > 1 and not any(k in name for k in sys.argv[1:]):
        continue
    mut = SRC.replace(a, b, 1)
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "m.c")
        so = os.path.join(d, "libm.so")
        open(c, "w").write(mut)
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", so, c, "-lm"])
        env = dict(os.environ, HSGN_ORACLE_LIB=so)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            os.path.join(ROOT, "tests", tf)],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        caught = r.returncode != 0
        first = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
        print(("CAUGHT " if caught else "MISSED ") + name + ("  <- " + first[0] if first else ""))
        ok &= caught
sys.exit(0 if ok else 1)
