TITLE Ih (BBP cortex) restated in the modlc subset
NEURON {
    SUFFIX Ih
    NONSPECIFIC_CURRENT ihcn
    RANGE gIhbar, gIh
}
PARAMETER {
    gIhbar = 0.00001 (S/cm2)
    ehcn = -45.0 (mV)
}
ASSIGNED {
    v (mV)
    ihcn (mA/cm2)
    gIh (S/cm2)
    mInf
    mTau
    mAlpha
    mBeta
}
STATE {
    m
}
BREAKPOINT {
    SOLVE states METHOD cnexp
    gIh = gIhbar*m
    ihcn = gIh*(v - ehcn)
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
    LOCAL u
    u = vm
    IF (u == -154.9) {
        u = u + 0.0001
    }
    mAlpha = 0.001*6.43*(u + 154.9)/(exp((u + 154.9)/11.9) - 1)
    mBeta = 0.001*193*exp(u/33.1)
    mInf = mAlpha/(mAlpha + mBeta)
    mTau = 1/(mAlpha + mBeta)
}
