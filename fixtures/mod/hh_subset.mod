TITLE hh restated in the modlc subset (no TABLE/UNITSOFF/THREADSAFE)
NEURON {
    SUFFIX hh
    USEION na READ ena WRITE ina
    USEION k READ ek WRITE ik
    NONSPECIFIC_CURRENT il
    RANGE gnabar, gkbar, gl, el
}
PARAMETER {
    gnabar = 0.12 (S/cm2)
    gkbar = 0.036 (S/cm2)
    gl = 0.0003 (S/cm2)
    el = -54.3 (mV)
}
ASSIGNED { v (mV) ina ik il minf hinf ninf mtau htau ntau }
STATE { m h n }
BREAKPOINT {
    SOLVE states METHOD cnexp
    ina = gnabar*m*m*m*h*(v - ena)
    ik = gkbar*n*n*n*n*(v - ek)
    il = gl*(v - el)
}
INITIAL { rates(v)
    m = minf
    h = hinf
    n = ninf }
DERIVATIVE states { rates(v)
    m' = (minf-m)/mtau
    h' = (hinf-h)/htau
    n' = (ninf-n)/ntau }
PROCEDURE rates(v (mV)) {
    LOCAL alpha, beta, sum, q10
    q10 = 3^((celsius - 6.3)/10)
    alpha = .1 * vtrap(-(v+40),10)
    beta = 4 * exp(-(v+65)/18)
    sum = alpha + beta
    mtau = 1/(q10*sum)
    minf = alpha/sum
    alpha = .07 * exp(-(v+65)/20)
    beta = 1 / (exp(-(v+35)/10) + 1)
    sum = alpha + beta
    htau = 1/(q10*sum)
    hinf = alpha/sum
    alpha = .01*vtrap(-(v+55),10)
    beta = .125*exp(-(v+65)/80)
    sum = alpha + beta
    ntau = 1/(q10*sum)
    ninf = alpha/sum
}
FUNCTION vtrap(x,y) {
    IF (fabs(x/y) < 1e-6) {
        vtrap = y*(1 - x/y/2)
    } ELSE {
        vtrap = x/(exp(x/y) - 1)
    }
}
