TITLE SKv3_1 (BBP cortex) restated in the modlc subset
NEURON {
    SUFFIX SKv3_1
    USEION k READ ek WRITE ik
    RANGE gSKv3_1bar, gSKv3_1
}
PARAMETER {
    gSKv3_1bar = 0.00001 (S/cm2)
}
ASSIGNED {
    v (mV)
    ek (mV)
    ik (mA/cm2)
    gSKv3_1 (S/cm2)
    mInf
    mTau
}
STATE {
    m
}
BREAKPOINT {
    SOLVE states METHOD cnexp
    gSKv3_1 = gSKv3_1bar*m
    ik = gSKv3_1*(v - ek)
}
DERIVATIVE states {
    rates(v)
    m' = (mInf - m)/mTau
}
INITIAL {
    rates(v)
    m = mInf
}
PROCEDURE rates(vm (mV)) {
    mInf = 1/(1 + exp(((vm - (18.700))/(-9.700))))
    mTau = 0.2*20.000/(1 + exp(((vm - (-46.560))/(-44.140))))
}
