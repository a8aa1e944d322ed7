"""Mutation sweep of the oracle (test infrastructure; CPU only): applies one plausible slip at a time (a dropped
term, a wrong sign, index, node or weight) to a COPY of oracle/ under /tmp and runs the oracle's pins (-m "not gpu")
against it.  A mutant that passes every pin is a hole in the pins (session 5 found six in oracle/lshape.py: the sign
of C in either row of slab_matrix and four slips of slab_load; pins L10 / L11 close them).  Mutants that change
nothing observable by design (e.g. the directional penalty length, equal to h_F in the default mode) are listed as
EQUIVALENT.

  python tools/mutate_oracle.py [-j 4] [name ...]      # table on stdout (profiles/r02/mutation_sweep_s5.txt)
"""
import argparse
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LSHAPE_TESTS = ["tests/test_oracle_lshape.py"]
BOX_TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_mg.py", "tests/test_oracle_ebe.py"]
EQUIVALENT = {"dir_pen_len": "h_D = h_F in the default penalty-length mode (reading R4)"}

LSHAPE = [
 ("sip_int_consistency_sign", '-0.5 * sg[i] * np.einsum("sq,rq,q->rs", kgn[j], ph[i], w)', '+0.5 * sg[i] * np.einsum("sq,rq,q->rs", kgn[j], ph[i], w)'),
 ("sip_int_symmetry_drop", '- 0.5 * sg[j] * np.einsum("sq,rq,q->rs", ph[j], kgn[i], w)', '- 0.0 * sg[j] * np.einsum("sq,rq,q->rs", ph[j], kgn[i], w)'),
 ("sip_int_pen_sign", 'pen * sg[i] * sg[j] * np.einsum("sq,rq,q->rs", ph[j], ph[i], w))\n        return Bf', 'pen * np.einsum("sq,rq,q->rs", ph[j], ph[i], w))\n        return Bf'),
 ("sip_int_avg_full", '-0.5 * sg[i]', '-1.0 * sg[i]'),
 ("sip_bnd_drop_sym", '- np.einsum("sq,rq,q->rs", php, Kgn, w)\n', '\n'),
 ("dir_pen_len", 'self.hF if kind == U_DIRICHLET else self.hD', 'self.hF'),
 ("dir_face_C_sign", 'C = self.p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, php, w)', 'C = -self.p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, php, w)'),
 ("dir_consistency_drop", 'A = (-np.einsum("Jq,Iq,q->IJ", snn, vn, w) - np.einsum("Jq,Iq,q->IJ", vn, snn, w)', 'A = (-np.einsum("Jq,Iq,q->IJ", snn, vn, w)'),
 ("vol_C_sign", 'C = -p["alpha"] * np.einsum("Jq,sq,q->sJ", div, php, w)', 'C = p["alpha"] * np.einsum("Jq,sq,q->sJ", div, php, w)'),
 ("interior_upper_face", 'if f % 2 == 1:                         # interior', 'if f % 2 == 0:                         # interior'),
 ("calK_C_sign", '[-S.C, None, S.B]', '[S.C, None, S.B]'),
 ("calK_CT", '[None, S.A, S.C.T]', '[None, S.A, -S.C.T]'),
 ("load_theta_drop", 'H.th[b] * np.sin(8.0 * np.pi * t) * fN', 'np.sin(8.0 * np.pi * t) * fN'),
 ("load_time_node", 't = t_prev + 0.5 * H.tau * (1.0 + H.t_hat[b])', 't = t_prev + H.tau * (1.0 + H.t_hat[b])'),
 ("load_freq", 'np.sin(8.0 * np.pi * t)', 'np.sin(4.0 * np.pi * t)'),
 ("load_row", 'o = lev.offset(b, 1, 0)\n        L[o:o + 3 * lev.nq]', 'o = lev.offset(b, 0, 0)\n        L[o:o + 3 * lev.nq]'),
 ("rhs_swap_UV", 'MU, MV, MP = S.Mr @ U, S.Mr @ V, S.Mc @ P', 'MU, MV, MP = S.Mr @ V, S.Mr @ U, S.Mc @ P'),
 ("rhs_first_block", 'o = k * lev.block\n    V = x_prev', 'o = 0 * lev.block\n    V = x_prev'),
 ("traction_sign", 'lev.nq + lev.cell_q[cid], -(phq', 'lev.nq + lev.cell_q[cid], (phq'),
 ("traction_comp", 'np.add.at(out, lev.nq + lev.cell_q[cid]', 'np.add.at(out, 2 * lev.nq + lev.cell_q[cid]'),
 ("traction_g", '32.0 * x * z - 18.0 * x - 16.0 * z + 10.0', '32.0 * x * z - 18.0 * x - 16.0 * z + 9.0'),
 ("goal_block", 'o = lev.k * lev.block\n    bu = bp', 'o = 0 * lev.block\n    bu = bp'),
 ("goal_comp", 'ux = x[o + lev.R + lev.cell_q[cid]]', 'ux = x[o + lev.R + lev.nq + lev.cell_q[cid]]'),
 ("goal_field", 'ux = x[o + lev.R + lev.cell_q[cid]]', 'ux = x[o + lev.cell_q[cid]]'),
 ("bc_z_neumann", 'if a == 2:\n            return U_DIRECTIONAL', 'if a == 2 and s == 0:\n            return U_DIRECTIONAL'),
 ("bc_x0", 'if a == 0 and s == 0:\n            return U_DIRECTIONAL', 'if a == 0 and s == 0:\n            return U_DIRICHLET'),
 ("bc_p_dir", 'return P_DIRICHLET if (a == 1 and s == 1 and c[1] == self.n[1] - 1)', 'return P_DIRICHLET if (a == 1 and s == 0 and c[1] == 0)'),
 ("vcycle_nopost", 'd = d + self.P[l] @ dc\n        return sm.smooth(b, d, self.jmax)', 'd = d + self.P[l] @ dc\n        return d'),
 ("vcycle_restrict_b", 'dc = self.vcycle(self.P[l].T @ r, l - 1)', 'dc = self.vcycle(self.P[l].T @ b, l - 1)'),
 ("prolong_Pp_parent", 'X = blocks[tuple(int(v % 2) for v in c)]', 'X = blocks[tuple(int((v + 1) % 2) for v in c)]'),
 ("load_time_node2", 't = t_prev + 0.5 * H.tau * (1.0 + H.t_hat[b])', 't = t_prev + 0.5 * H.tau * (1.0 + H.t_hat[lev.k - b])'),
 ("load_cos", 'np.sin(8.0 * np.pi * t)', 'np.cos(8.0 * np.pi * t)'),
 ("patch_drop_last_p", 'idx.append(lev.offset(m, 2) + pn)', 'idx.append(lev.offset(m, 2) + pn[:-1])'),
]
LOADS = [
 ("f_dtt", 'rho * sy.diff(u[i], t, 2)', 'rho * sy.diff(u[i], t, 1)'),
 ("f_gradp_sign", '+ alpha * sy.diff(p, X[i]) for i in range(d)]', '- alpha * sy.diff(p, X[i]) for i in range(d)]'),
 ("g_div_sign", 'g = c0 * sy.diff(p, t) + alpha * sum(', 'g = c0 * sy.diff(p, t) - alpha * sum('),
 ("g_K_sign", '- sum(sy.diff(Kgp[i], X[i]) for i in range(d))', '+ sum(sy.diff(Kgp[i], X[i]) for i in range(d))'),
 ("trac_weight", 'w = _tensor_weights(wts, float(np.prod(lev.h)) / lev.h[a])\n    loc = phq @ w', 'w = _tensor_weights(wts, float(np.prod(lev.h)))\n    loc = phq @ w'),
 ("trac_side", 'sel = cells[:, a] == (0 if s == 0 else lev.n[a] - 1)\n    qn = D[sel]', 'sel = cells[:, a] == (0 if s == 1 else lev.n[a] - 1)\n    qn = D[sel]'),
 ("trac_comp", 'np.add.at(F, comp * lev.nq + qn, amplitude * loc[None, :])', 'np.add.at(F, ((comp + 1) % d) * lev.nq + qn, amplitude * loc[None, :])'),
 ("rhs_theta_F", 'Rv[o + lev.R: o + 2 * lev.R] += th[b] * Floads[b]', 'Rv[o + lev.R: o + 2 * lev.R] += Floads[b]'),
 ("rhs_theta_G", 'Rv[o + 2 * lev.R: o + lev.block] += th[b] * Gloads[b]', 'Rv[o + 2 * lev.R: o + lev.block] += Gloads[b]'),
 ("rhs_swap", 'Rv[o: o + lev.R] = chi_m1[b] * MU\n        Rv[o + lev.R: o + 2 * lev.R] = chi_m1[b] * MV', 'Rv[o: o + lev.R] = chi_m1[b] * MV\n        Rv[o + lev.R: o + 2 * lev.R] = chi_m1[b] * MU'),
 ("goal_nrm", 'nrm = 1.0 if s == 1 else -1.0', 'nrm = 1.0'),
 ("init_v", 'V = sol.v(xq, t0).T.ravel()', 'V = 0 * sol.v(xq, t0).T.ravel()'),
]
ELEMENT = [
 ("e_CT_sign", 'blk[sU, sP] = th[b] * C.T', 'blk[sU, sP] = -th[b] * C.T'),
 ("e_C_sign", 'blk[sP, sV] = -th[b] * C', 'blk[sP, sV] = th[b] * C'),
 ("e_VV_sign", 'blk[sV, sV] = -th[b] * Mr', 'blk[sV, sV] = th[b] * Mr'),
 ("e_nitsche_sym", '- np.einsum("Jqa,Iqa,q->IJ", Vf, sn, fw)      # -<w, sigma(chi) n>', '- 0 * np.einsum("Jqa,Iqa,q->IJ", Vf, sn, fw)'),
 ("e_Cface_sign", 'C += p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, fphp, fw)', 'C -= p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, fphp, fw)'),
 ("e_Cface_drop", 'C += p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, fphp, fw)', 'C += 0 * np.einsum("Jq,sq,q->sJ", vn, fphp, fw)'),
 ("e_normal", 'n[a] = -1.0 if s == 0 else 1.0', 'n[a] = 1.0'),
 ("e_hF_edge", 'return self.vol                 # |K|_d, P:L205 (reading A6)', 'return float(self.h[0])'),
 ("e_B_sym_drop", '- np.einsum("sq,rq,q->rs", fphp, Kgn, fw)', '- 0 * np.einsum("sq,rq,q->rs", fphp, Kgn, fw)'),
 ("e_lam2", 'sig[:, :, i, i] += lam * tr', 'sig[:, :, i, i] += 2 * lam * tr'),
 ("e_ds_sign", 'blk[sP, sU] = -T[b, a] * C', 'blk[sP, sU] = T[b, a] * C'),
 ("e_pen_a_b", 'pen = ga / self.hF(f)', 'pen = gb / self.hF(f)'),
]
VANKA = [
 ("v_no_averaging", 'return d + self.omega * z / self.P.p', 'return d + self.omega * z'),
 ("v_unscale", 'return inv * s[:, None] * s[None, :]', 'return inv * s[:, None]'),
 ("v_post_from_zero", 'd = np.zeros_like(b) if d is None else d.copy()', 'd = np.zeros_like(b)'),
 ("v_class_rep_inverse", 'Y = r[Z] @ self.inv[mem[0]].T', 'Y = r[Z] @ self.inv[mem[0]]'),
]
TRANSFER = [
 ("t_child_offset", 'xf = 0.5 * ((cf % 2) + nodes)', 'xf = 0.5 * (((cf + 1) % 2) + nodes)'),
 ("t_pressure_degree", 'Pp = kron_axes(r - 1)', 'Pp = kron_axes(r - 1) * 2.0'),
 ("t_transposed_weights", 'P[deg * cf + i, deg * cc + j] = V[j, i]', 'P[deg * cf + i, deg * cc + j] = V[i, j]'),
]
TEMPORAL = [
 ("tm_T_transposed", 'T[b, a] = w[b] * D[a, b] + Vm1[a] * Vm1[b]', 'T[b, a] = w[b] * D[b, a] + Vm1[a] * Vm1[b]'),
 ("tm_no_jump", 'T[b, a] = w[b] * D[a, b] + Vm1[a] * Vm1[b]', 'T[b, a] = w[b] * D[a, b]'),
 ("tm_weight_index", 'T[b, a] = w[b] * D[a, b] + Vm1[a] * Vm1[b]', 'T[b, a] = w[a] * D[a, b] + Vm1[a] * Vm1[b]'),
]
MG = [
 ("mg_no_post", 'd = d + self.P[l] @ dc\n        return sm.smooth(b, d, self.jmax, self.colored, self.overwrite)', 'd = d + self.P[l] @ dc\n        return d'),
 ("mg_restrict_b", 'dc = self.vcycle(self.P[l].T @ r, l - 1)', 'dc = self.vcycle(self.P[l].T @ b, l - 1)'),
 ("mg_correction_sign", 'd = d + self.P[l] @ dc', 'd = d - self.P[l] @ dc'),
]
GROUPS = [("oracle/lshape.py", LSHAPE, LSHAPE_TESTS), ("oracle/loads.py", LOADS, BOX_TESTS),
          ("oracle/element.py", ELEMENT, BOX_TESTS), ("oracle/vanka.py", VANKA, BOX_TESTS),
          ("oracle/transfer.py", TRANSFER, BOX_TESTS), ("oracle/temporal.py", TEMPORAL, BOX_TESTS),
          ("oracle/mg.py", MG, BOX_TESTS)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=4)
    ap.add_argument("names", nargs="*")
    a = ap.parse_args()
    jobs = []
    for path, muts, tests in GROUPS:
        src = open(os.path.join(ROOT, path)).read()
        for name, old, new in muts:
            if a.names and name not in a.names:
                continue
            assert src.count(old) == 1, (name, "pattern matches %d times" % src.count(old))
            d = "/tmp/stgmg_mut_" + name
            shutil.rmtree(d, ignore_errors=True)
            os.makedirs(d)
            for sub in ("oracle", "tests", "stgmg_inputs"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub))
            with open(os.path.join(d, path), "w") as f:
                f.write(src.replace(old, new))
            jobs.append((path, name, d, tests))
    survivors = 0
    for i in range(0, len(jobs), a.j):
        procs = []
        for path, name, d, tests in jobs[i:i + a.j]:
            log = open(os.path.join(d, "out.log"), "w")
            procs.append((path, name, d, subprocess.Popen(
                ["python", "-m", "pytest"] + tests + ["-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider"],
                cwd=d, stdout=log, stderr=subprocess.STDOUT)))
        for path, name, d, p in procs:
            p.wait()
            lines = open(os.path.join(d, "out.log")).read().strip().splitlines()
            failed = [ln for ln in lines if ln.startswith("FAILED")]
            if p.returncode:
                verdict = "KILLED by " + (failed[0].split("::")[1].split(" ")[0] if failed else "?")
            elif name in EQUIVALENT:
                verdict = "EQUIVALENT (" + EQUIVALENT[name] + ")"
            else:
                verdict = "SURVIVED"
                survivors += 1
            print("%-18s %-24s %s" % (path, name, verdict), flush=True)
            shutil.rmtree(d, ignore_errors=True)
    print("%d mutants, %d survivors" % (len(jobs), survivors))
    return 1 if survivors else 0


if __name__ == "__main__":
    raise SystemExit(main())
