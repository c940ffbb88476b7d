TITLE K_Pst (BBP cortex) restated in the modlc subset
NEURON {
    SUFFIX K_Pst
    USEION k READ ek WRITE ik
    RANGE gK_Pstbar, gK_Pst
}
PARAMETER {
    gK_Pstbar = 0.00001 (S/cm2)
}
ASSIGNED {
    v (mV)
    ek (mV)
    ik (mA/cm2)
    gK_Pst (S/cm2)
    mInf
    mTau
    hInf
    hTau
}
STATE {
    m
    h
}
BREAKPOINT {
    SOLVE states METHOD cnexp
    gK_Pst = gK_Pstbar*m*m*h
    ik = gK_Pst*(v - ek)
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
    LOCAL qt, u
    qt = 2.3^((34 - 21)/10)
    u = vm + 10
    mInf = 1/(1 + exp(-(u + 1)/12))
    IF (u < -50) {
        mTau = (1.25 + 175.03*exp(-u*-0.026))/qt
    } ELSE {
        mTau = (1.25 + 13*exp(-u*0.026))/qt
    }
    hInf = 1/(1 + exp(-(u + 54)/-11))
    hTau = (360 + (1010 + 24*(u + 55))*exp(-((u + 75)/48)^2))/qt
}
