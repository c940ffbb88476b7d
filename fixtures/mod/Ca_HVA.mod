TITLE Ca_HVA (BBP cortex) restated in the modlc subset
NEURON {
    SUFFIX Ca_HVA
    USEION ca READ eca WRITE ica
    RANGE gCa_HVAbar, gCa_HVA
}
PARAMETER {
    gCa_HVAbar = 0.00001 (S/cm2)
}
ASSIGNED {
    v (mV)
    eca (mV)
    ica (mA/cm2)
    gCa_HVA (S/cm2)
    mInf
    mTau
    mAlpha
    mBeta
    hInf
    hTau
    hAlpha
    hBeta
}
STATE {
    m
    h
}
BREAKPOINT {
    SOLVE states METHOD cnexp
    gCa_HVA = gCa_HVAbar*m*m*h
    ica = gCa_HVA*(v - eca)
}
DERIVATIVE states {
    rates(v)
    m' = (mInf - m)/mTau
    h' = (hInf - h)/hTau
}
INITIAL {
    rates(v)
    m = mInf
    h = hInf
}
PROCEDURE rates(vm (mV)) {
    LOCAL u
    u = vm
    IF (u == -27) {
        u = u + 0.0001
    }
    mAlpha = (0.055*(-27 - u))/(exp((-27 - u)/3.8) - 1)
    mBeta = (0.94*exp((-75 - u)/17))
    mInf = mAlpha/(mAlpha + mBeta)
    mTau = 1/(mAlpha + mBeta)
    hAlpha = (0.000457*exp((-13 - u)/50))
    hBeta = (0.0065/(exp((-u - 15)/28) + 1))
    hInf = hAlpha/(hAlpha + hBeta)
    hTau = 1/(hAlpha + hBeta)
}
