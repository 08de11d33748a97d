"""Oracle for the SFB-vs-AllReduce selector and the closed-form communication volumes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Exact arithmetic throughout: Python ints for
byte counts and decisions, fractions.Fraction for times, so that no floating-point rounding can
decide anything.

Sources (P:n = PAPER.md line n, S:n = SPEC.md line n):
  * SFB volume (Fig. 5): the gradient H2 x H1 is replaced by the sufficient factors,
    2(H2*B + B*H1) elements at D = 2.
  * SFB ILP (Table "Notation in SFB Optimization" P:578-600):
        min (D-1) sum_i a_i T_i + D(D-1) sum_(j,i) b_ji L_ji / tau - 2 a_g (D-1)/D L_gl / tau
    specialised to one Dense-layer MatMul (reading R4b): V = {g, l}, cut = {x, grad},
    alpha_l = 1, so alpha_g = 1 costs
        (D-1) T_g + D(D-1)(L_x + L_grad)/tau - 2 (D-1)/D L_gl / tau
    and SFB is chosen iff that is < 0 (tie -> AllReduce).
  * Ring AllReduce time 2(D-1)/D * L / tau.
  * Linear compute model: T_g = 2 M N B / F.
  * north_star's byte rule: n B (M+N) e_w (gathered factors) vs 2 M N (n-1)/n e_g (ring AR).

Three readings of the SFB communication term, because the paper's ILP, north_star and the
physical NVSwitch traffic disagree for n > 2 (R2):
    RULE_NORTHSTAR  : n   * S / tau       (gathered factor bytes; north_star literal)  [default]
    RULE_PAPER_ILP  : n(n-1) * S / tau    (the ILP's D(D-1) broadcast term)
    RULE_WIRE       : (n-1) * S / tau     (bytes each rank receives in an all-gather)
with S = B (M+N) e_w the per-replica factor bytes (L_x + L_grad, R3) and G = M N e_g.
"""
from fractions import Fraction

RULE_NORTHSTAR = 0
RULE_PAPER_ILP = 1
RULE_WIRE = 2

CHOICE_ALLREDUCE = 0
CHOICE_SFB = 1
CHOICE_NONE = 2
CHOICE_PS = 3            # Replicate with PS, profiled selector only


def sfb_elements_fig5(H1, H2, B):
    """Total elements communicated by SFB for one Dense layer at D = 2: 2(H2*B + B*H1)."""
    return 2 * (H2 * B + B * H1)


def gradient_elements(H1, H2):
    """Elements of the gradient the SFB replaces: H2 x H1."""
    return H2 * H1


def sfb_gathered_bytes(n, B, M, N, e_w):
    """north_star's SFB bytes: n * B * (M + N) * e_w — the factor buffer every replica ends with."""
    return n * B * (M + N) * e_w


def allgather_ingress_bytes(n, B, M, N, e_w):
    """Bytes each replica receives in the factor all-gather: (n-1) * B * (M+N) * e_w."""
    return (n - 1) * B * (M + N) * e_w


def ring_allreduce_bytes(n, M, N, e_g):
    """Ring AllReduce traffic per rank 2 (n-1)/n * M N e_g, as an exact Fraction."""
    return Fraction(2 * (n - 1) * M * N * e_g, n)


def ring_allreduce_time(D, size_bytes, tau):
    """SPEC predict_allreduce analytic fallback: 2(D-1)/D * size / tau seconds; D = 1 -> 0."""
    if D <= 1:
        return Fraction(0)
    return Fraction(2 * (D - 1) * size_bytes, D) / Fraction(tau)


def ilp_objective(D, T_g, cut_bytes, L_gl, tau, alpha_g=1):
    """Objective of the specialised SFB ILP for alpha_g in {0, 1}, b = alpha_g on the cut
    (constraint 2, with replicated producers alpha_j = 0). Exact Fraction seconds."""
    if alpha_g == 0:
        return Fraction(0)
    T_g = Fraction(T_g)
    return ((D - 1) * T_g + D * (D - 1) * Fraction(cut_bytes) / Fraction(tau)
            - 2 * Fraction(D - 1, D) * Fraction(L_gl) / Fraction(tau))


def sfb_cost_terms(layer, topo):
    """(sfb_seconds, allreduce_seconds) as exact Fractions for one layer under topo's rule.
    layer: dict(M, N, B, e_w, e_g); topo: dict(n, tau, F, rule). F = 0 drops the compute term."""
    n, tau, F, rule = topo["n"], topo["tau"], topo["F"], topo.get("rule", RULE_NORTHSTAR)
    M, N, B, e_w, e_g = layer["M"], layer["N"], layer["B"], layer["e_w"], layer["e_g"]
    S = B * (M + N) * e_w
    G = M * N * e_g
    mult = {RULE_NORTHSTAR: n, RULE_PAPER_ILP: n * (n - 1), RULE_WIRE: n - 1}[rule]
    compute = Fraction((n - 1) * 2 * M * N * B, F) if F else Fraction(0)
    sfb = compute + Fraction(mult * S, tau)
    ar = Fraction(2 * (n - 1) * G, n * tau)
    return sfb, ar


def select(layer, topo):
    """Per-layer decision ("needs to be examined for each gradient").
    n = 1 -> NONE (S:476 NotApplicable for D < 2). SFB iff its cost is strictly lower; a tie keeps
    AllReduce ("objective >= 0 -> strategy unchanged")."""
    if topo["n"] <= 1:
        return CHOICE_NONE
    sfb, ar = sfb_cost_terms(layer, topo)
    return CHOICE_SFB if sfb < ar else CHOICE_ALLREDUCE


def select_integer_form(layer, topo):
    """The same decision written as the cleared-denominator integer inequality the library
    evaluates (multiply both sides by n * tau * F > 0; R4c). Python ints are exact."""
    n, tau, F, rule = topo["n"], topo["tau"], topo["F"], topo.get("rule", RULE_NORTHSTAR)
    if n <= 1:
        return CHOICE_NONE
    M, N, B, e_w, e_g = layer["M"], layer["N"], layer["B"], layer["e_w"], layer["e_g"]
    S = B * (M + N) * e_w
    G = M * N * e_g
    mult = {RULE_NORTHSTAR: n, RULE_PAPER_ILP: n * (n - 1), RULE_WIRE: n - 1}[rule]
    if F:
        lhs = n * (n - 1) * 2 * M * N * B * tau + n * mult * S * F
        rhs = 2 * (n - 1) * G * F
    else:
        lhs = n * mult * S
        rhs = 2 * (n - 1) * G
    return CHOICE_SFB if lhs < rhs else CHOICE_ALLREDUCE


# ---------------------------------------------------------------------------------------------
# Profiled selector (the paper's profiler: "Segmented linear regression models are built
# for GRPC transfer and for AllReduce communication"; SPEC fit_comm S:197-205 realises it as exact
# piecewise-linear interpolation between consecutive profiled sizes, extended by the first / last
# segment). Times in integer ns with floor rounding, clamped at 0, so the library's integer
# evaluation can be compared decision for decision.
# ---------------------------------------------------------------------------------------------
def curve_ns(points, x):
    """points: [(bytes, ns), ...] with strictly increasing bytes (>= 2 points)."""
    i = 0
    while i + 2 < len(points) and x > points[i + 1][0]:
        i += 1
    (b0, t0), (b1, t1) = points[i], points[i + 1]
    t = t0 + ((x - b0) * (t1 - t0)) // (b1 - b0)       # Python // is floor division
    return max(t, 0)


def select_profiled(layer, n, gather_pts, allreduce_pts, F=0, ps_pts=None, recon_ns=None,
                    local_ns=None):
    """SFB iff gather((n-1) S) + floor((n-1) 2MNB 1e9 / F) < allreduce(G); ties -> AllReduce.
    With a PS curve ("Replicate with PS"): PS iff ps(G) is strictly below both
    (ties: AllReduce, then SFB). With measured op times (the paper's profiler) the
    compute term is the measured one: SFB = gather + recon_ns, AllReduce = local_ns + ar(G),
    PS = local_ns + ps(G)."""
    if n <= 1:
        return CHOICE_NONE
    M, N, B, e_w, e_g = layer["M"], layer["N"], layer["B"], layer["e_w"], layer["e_g"]
    S = B * (M + N) * e_w
    G = M * N * e_g
    t_sfb = curve_ns(gather_pts, (n - 1) * S)
    t_local = 0
    if recon_ns is not None:
        t_sfb += recon_ns
        t_local = local_ns
    elif F:
        t_sfb += ((n - 1) * 2 * M * N * B * 10 ** 9) // F
    costs = [(t_local + curve_ns(allreduce_pts, G), 0, CHOICE_ALLREDUCE), (t_sfb, 1, CHOICE_SFB)]
    if ps_pts:
        costs.append((t_local + curve_ns(ps_pts, G), 2, CHOICE_PS))
    return min(costs)[2]


# ---------------------------------------------------------------------------------------------
# The general SFB ILP (SPEC solve_bruteforce S:490-495), by exhaustive enumeration.
#   min (D-1) sum_i a_i T_i + D(D-1) sum_{(j,i) in E} b_ji L_ji / tau - 2 a_g (D-1)/D L_gl / tau
#   s.t. a_k <= sum_{(k,i) in E} a_i  for k in V \ {l};  b_ji >= a_i - a_j;  a, b binary.
# Readings (DESIGN R20): a_l = 1 and T_l excluded; producers outside the group have
# a = 0 (src = -1); edges into l are not cut candidates (l runs on every replica either way; the
# gradient's own synchronisation is the third term); b_ji = max(0, a_i - a_j), the cheapest
# feasible cut. Ties: the assignment duplicating the fewest ops wins (then the lexicographically
# smallest a vector, which ilp_bruteforce reports as `ambiguous` — the minimal optimum is unique
# because minimum cuts form a lattice, DESIGN R20).
# ---------------------------------------------------------------------------------------------
def ilp_eval(inst, alpha):
    """Exact objective (Fraction seconds) of assignment `alpha` (list of 0/1, alpha[l] == 1), or
    None if it violates constraint 1."""
    V, l, g = inst["num_ops"], inst["l"], inst["g"]
    D, tau = inst["D"], inst["tau"]
    edges = inst["edges"]                     # [(src or -1, dst, bytes)]
    for k in range(V):
        if k == l or not alpha[k]:
            continue
        if not any(alpha[i] for (j, i, _) in edges if j == k):
            return None
    obj = Fraction(0)
    for i in range(V):
        if i != l and alpha[i]:
            obj += Fraction((D - 1) * inst["op_ns"][i], 10 ** 9)
    for (j, i, L) in edges:
        if i == l:
            continue
        aj = alpha[j] if j >= 0 else 0
        if alpha[i] - aj > 0:
            obj += Fraction(D * (D - 1) * L, tau)
    if alpha[g]:
        obj -= 2 * Fraction(D - 1, D) * Fraction(inst["grad_bytes"], tau)
    return obj


def ilp_bruteforce(inst):
    """(objective, alpha, ambiguous) minimising over all 2^(|V|-1) assignments with alpha_l = 1.
    `ambiguous` is True when another optimum duplicates equally few ops."""
    V, l = inst["num_ops"], inst["l"]
    free = [k for k in range(V) if k != l]
    best, ambiguous = None, False
    for mask in range(1 << len(free)):
        alpha = [0] * V
        alpha[l] = 1
        for b, k in enumerate(free):
            alpha[k] = (mask >> b) & 1
        obj = ilp_eval(inst, alpha)
        if obj is None:
            continue
        key = (obj, sum(alpha))
        if best is None or key < (best[0], sum(best[1])):
            best, ambiguous = (obj, alpha), False
        elif key == (best[0], sum(best[1])):
            ambiguous = True
    return best[0], best[1], ambiguous
