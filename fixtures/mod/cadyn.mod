TITLE CaDynamics_E2-style accumulation (FARADAY inlined as a literal)
NEURON { SUFFIX CaDynamics_E2
    USEION ca READ ica WRITE cai
    RANGE decay, gamma, minCai, depth }
PARAMETER { gamma = 0.05 decay = 80 depth = 0.1 minCai = 1e-4 }
ASSIGNED { v (mV) ica }
STATE { cai }
BREAKPOINT { SOLVE states METHOD cnexp }
INITIAL { cai = minCai }
DERIVATIVE states {
    cai' = -(10000)*(ica*gamma/(2*96485.3329*depth)) - (cai - minCai)/decay
}
