TITLE kernel-written GLOBALs and slot-based exponentials (backend regression fixture)
COMMENT
Not a BASELINE mechanism: exercises code-generation hazards.
* cnt is a GLOBAL the kernels update uniformly from its own value (cnt = cnt + 1,
  in nrn_state and in nrn_cur): every instance must see the value the launch
  started with, and the numeric-conductance v+h pass keeps its GLOBAL write
  (the reference restores arrays, not scalars, modlc/interp.py:498-507).
* y reads exp(0.01*s) before and after the slot s is reassigned: an exp cached
  on the slot's old value must not be reused.
ENDCOMMENT
NEURON {
    SUFFIX rwglobal
    NONSPECIFIC_CURRENT i
    RANGE gbar, s, y
    GLOBAL cnt
}
PARAMETER {
    gbar = 0.002
}
ASSIGNED {
    v (mV)
    i
    s
    y
    cnt
}
STATE {
    u
}
BREAKPOINT {
    SOLVE du METHOD cnexp
    cnt = cnt + 1
    i = gbar*u*exp(v/50)*(v + 70)*(1 + 1e-6*cnt)
}
INITIAL {
    cnt = 0
    u = 0.3
    s = 1
}
DERIVATIVE du {
    y = exp(0.01*s)
    s = v
    y = y + exp(0.01*s)
    cnt = cnt + 1
    u' = (0.5 + 0.001*y - u)/(5 + 0.01*cnt)
}
