TITLE ProbAMPANMDA_EMS restated in the modlc subset (AMPA + NMDA double exponential, Mg block)
COMMENT
The stock BBP synapse drives its states from NET_RECEIVE and RANDOM streams,
which the reference front-end rejects (modlc/lexer.py:62-89). This restatement
keeps the per-timestep nrn_state/nrn_cur arithmetic: four cnexp decays, the
Jahr-Stevens Mg block and the non-ohmic current that forces the two-point
numeric conductance. An event of weight w0 is applied at INITIAL so that the
trajectories are not identically zero.
ENDCOMMENT
NEURON {
    POINT_PROCESS ProbAMPANMDA_EMS
    RANGE tau_r_AMPA, tau_d_AMPA, tau_r_NMDA, tau_d_NMDA
    RANGE Use, u0, Dep, Fac, Nrrp, w0
    RANGE i, i_AMPA, i_NMDA, g_AMPA, g_NMDA, g, e, NMDA_ratio, gmax, mg
    NONSPECIFIC_CURRENT i
}
PARAMETER {
    tau_r_AMPA = 0.2 (ms)
    tau_d_AMPA = 1.7 (ms)
    tau_r_NMDA = 0.29 (ms)
    tau_d_NMDA = 43 (ms)
    Use = 1.0 (1)
    Dep = 100 (ms)
    Fac = 10 (ms)
    e = 0 (mV)
    mg = 1 (mM)
    gmax = .001 (uS)
    u0 = 0
    Nrrp = 1 (1)
    NMDA_ratio = 0.71 (1)
    w0 = 1 (1)
}
ASSIGNED {
    v (mV)
    i (nA)
    i_AMPA (nA)
    i_NMDA (nA)
    g_AMPA (uS)
    g_NMDA (uS)
    g (uS)
    factor_AMPA
    factor_NMDA
    mggate
}
STATE {
    A_AMPA
    B_AMPA
    A_NMDA
    B_NMDA
}
INITIAL {
    LOCAL tp_AMPA, tp_NMDA
    tp_AMPA = (tau_r_AMPA*tau_d_AMPA)/(tau_d_AMPA - tau_r_AMPA)*log(tau_d_AMPA/tau_r_AMPA)
    tp_NMDA = (tau_r_NMDA*tau_d_NMDA)/(tau_d_NMDA - tau_r_NMDA)*log(tau_d_NMDA/tau_r_NMDA)
    factor_AMPA = -exp(-tp_AMPA/tau_r_AMPA) + exp(-tp_AMPA/tau_d_AMPA)
    factor_AMPA = 1/factor_AMPA
    factor_NMDA = -exp(-tp_NMDA/tau_r_NMDA) + exp(-tp_NMDA/tau_d_NMDA)
    factor_NMDA = 1/factor_NMDA
    A_AMPA = w0*factor_AMPA
    B_AMPA = w0*factor_AMPA
    A_NMDA = w0*NMDA_ratio*factor_NMDA
    B_NMDA = w0*NMDA_ratio*factor_NMDA
}
BREAKPOINT {
    SOLVE state METHOD cnexp
    mggate = 1/(1 + exp(0.062*(-v))*(mg/3.57))
    g_AMPA = gmax*(B_AMPA - A_AMPA)
    g_NMDA = gmax*(B_NMDA - A_NMDA)*mggate
    g = g_AMPA + g_NMDA
    i_AMPA = g_AMPA*(v - e)
    i_NMDA = g_NMDA*(v - e)
    i = i_AMPA + i_NMDA
}
DERIVATIVE state {
    A_AMPA' = -A_AMPA/tau_r_AMPA
    B_AMPA' = -B_AMPA/tau_d_AMPA
    A_NMDA' = -A_NMDA/tau_r_NMDA
    B_NMDA' = -B_NMDA/tau_d_NMDA
}
