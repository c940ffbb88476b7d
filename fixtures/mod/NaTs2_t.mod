TITLE NaTs2_t (BBP cortex) restated in the modlc subset
COMMENT
Original uses UNITSOFF and assigns v inside rates() to dodge 0/0 at the
singular points; here the guard acts on a LOCAL copy of the formal.
ENDCOMMENT
NEURON {
    SUFFIX NaTs2_t
    USEION na READ ena WRITE ina
    RANGE gNaTs2_tbar, gNaTs2_t
}
PARAMETER {
    gNaTs2_tbar = 0.00001 (S/cm2)
}
ASSIGNED {
    v (mV)
    ena (mV)
    ina (mA/cm2)
    gNaTs2_t (S/cm2)
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
    gNaTs2_t = gNaTs2_tbar*m*m*m*h
    ina = gNaTs2_t*(v - ena)
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
    qt = 2.3^((celsius - 21)/10)
    u = vm
    IF (u == -32) {
        u = u + 0.0001
    }
    mAlpha = (0.182*(u - -32))/(1 - (exp(-(u - -32)/6)))
    mBeta = (0.124*(-u - 32))/(1 - (exp(-(-u - 32)/6)))
    mInf = mAlpha/(mAlpha + mBeta)
    mTau = (1/(mAlpha + mBeta))/qt
    u = vm
    IF (u == -60) {
        u = u + 0.0001
    }
    hAlpha = (-0.015*(u - -60))/(1 - (exp((u - -60)/6)))
    hBeta = (-0.015*(-u - 60))/(1 - (exp((-u - 60)/6)))
    hInf = hAlpha/(hAlpha + hBeta)
    hTau = (1/(hAlpha + hBeta))/qt
}
